// geoshoot/shooting.hpp -- shooting, objective, adjoint gradient and warp
// (reference shooting.hpp:26-86). The whole time loop runs on the device:
// trajectory, per-step trees and adjoints stay in HBM; only the report, the
// gradient (and, on request, the trajectory) come back.
#pragma once

#include <vector>

#include "geoshoot/bh_kernel.hpp"
#include "geoshoot/core.hpp"
#include "geoshoot/kernel_exact.hpp"

namespace geoshoot {

struct AdjointState {
  std::vector<Vec3> alpha;
  std::vector<Vec3> beta;
};

struct ObjectiveReport {
  double energy = 0.0;
  double attachment = 0.0;
  double total = 0.0;
  double residual_sse = 0.0;
};

struct EvalStats {
  double tree_build_ms = 0.0;
  double forward_ms = 0.0;
  double backward_ms = 0.0;
  TraversalStats traversal;
  std::uint64_t traversal_queries = 0;
  void merge(const EvalStats& o) {
    tree_build_ms += o.tree_build_ms;
    forward_ms += o.forward_ms;
    backward_ms += o.backward_ms;
    traversal.merge(o.traversal);
    traversal_queries += o.traversal_queries;
  }
};

GeodesicTrajectory shoot_forward(const PointSet& q0, const MomentumSet& p0,
                                 const ShootingConfig& config);
ObjectiveReport objective(const PointSet& q0, const MomentumSet& p0, const PointSet& target,
                          const ShootingConfig& config);
std::vector<Vec3> backward_gradient(const GeodesicTrajectory& trajectory, const PointSet& target,
                                    const ShootingConfig& config);
PointSet warp_points(const GeodesicTrajectory& trajectory, const PointSet& x,
                     const ShootingConfig& config);

struct Evaluation {
  ObjectiveReport report;
  std::vector<Vec3> gradient;
  EvalStats stats;
};

Evaluation evaluate(const PointSet& q0, const MomentumSet& p0, const PointSet& target,
                    const ShootingConfig& config, int threads = 0);

}  // namespace geoshoot
