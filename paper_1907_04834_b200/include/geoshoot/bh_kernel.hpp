// geoshoot/bh_kernel.hpp -- Barnes-Hut sums (reference bh_kernel.hpp:28-99),
// computed by the warp-cooperative sm_100a traversal. Same gate (tight-box
// min distance > threshold, leaf first), same centroid aggregates, same
// per-query statistics as the reference.
#pragma once

#include <cstdint>

#include "geoshoot/kernel_exact.hpp"
#include "geoshoot/octree.hpp"

namespace geoshoot {

struct TraversalStats {
  std::uint64_t direct_interactions = 0;
  std::uint64_t approximated_interactions = 0;
  std::uint64_t nodes_visited = 0;
  void merge(const TraversalStats& o) {
    direct_interactions += o.direct_interactions;
    approximated_interactions += o.approximated_interactions;
    nodes_visited += o.nodes_visited;
  }
};

/// The reference's compile-time GEOSHOOT_BH_LITERAL_MEAN_DOT switch
/// (bh_kernel.cpp:19-26: aggregate dot scale 1/count) as a runtime setting of
/// this thread's tree-level Barnes-Hut calls. Shooting uses
/// ShootingConfig::literal_mean_dot.
void set_bh_literal_mean_dot(bool enable);

struct BhVelocity {
  Vec3 velocity;
  TraversalStats stats;
};
BhVelocity bh_velocity(const Octree& tree, const Vec3& x, double sigma, double threshold);

struct BhPointGradients {
  Vec3 dH_dp;
  Vec3 dH_dq;
};
BhPointGradients bh_point_gradients(const Octree& tree, const Vec3& x, const Vec3& px, double sigma,
                                    double threshold, TraversalStats* stats = nullptr);

struct BhPointHessianProducts {
  Vec3 pq_alpha;
  Vec3 pp_alpha;
  Vec3 qq_beta;
  Vec3 qp_beta;
};
BhPointHessianProducts bh_point_hessian_products(const Octree& tree, const Vec3& qi,
                                                 const Vec3& pi, const Vec3& alpha_i,
                                                 const Vec3& beta_i,
                                                 const std::vector<Vec3>& alpha,
                                                 const std::vector<Vec3>& beta, double sigma,
                                                 double threshold, TraversalStats* stats = nullptr);

double bh_hamiltonian(const Octree& tree, const PointSet& q, const MomentumSet& p, double sigma,
                      double threshold, TraversalStats* stats = nullptr);
HamiltonianGradients bh_hamiltonian_gradients(const Octree& tree, const PointSet& q,
                                              const MomentumSet& p, double sigma, double threshold,
                                              TraversalStats* stats = nullptr);
HessianProducts bh_hessian_products(const Octree& tree, const PointSet& q, const MomentumSet& p,
                                    const std::vector<Vec3>& alpha, const std::vector<Vec3>& beta,
                                    double sigma, double threshold, TraversalStats* stats = nullptr);

}  // namespace geoshoot
