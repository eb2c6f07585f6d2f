// geoshoot/kernel_exact.hpp -- exact O(N^2) kernel sums (reference
// kernel_exact.hpp:37-80), computed by the sm_100a all-pairs kernels.
// Convention (reference kernel_exact.hpp:22-28): H = sum_ij (p_i.p_j) G_ij with
// no 1/2 and G(0) = 1, hence dH/dp_i = 2 sum_j G_ij p_j.
#pragma once

#include <vector>

#include "geoshoot/core.hpp"

namespace geoshoot {

inline double gaussian(double r, double sigma) {
  const double u = r / sigma;
  return std::exp(-0.5 * u * u);
}

inline constexpr double flow_velocity_factor = 2.0;

struct HamiltonianGradients {
  std::vector<Vec3> dH_dp;
  std::vector<Vec3> dH_dq;
};

double hamiltonian(const PointSet& q, const MomentumSet& p, double sigma);
double hamiltonian_with_gradients(const PointSet& q, const MomentumSet& p, double sigma,
                                  HamiltonianGradients& out);
HamiltonianGradients hamiltonian_gradients(const PointSet& q, const MomentumSet& p, double sigma);
std::vector<Vec3> exact_velocity(const PointSet& q_eval, const PointSet& q_src,
                                 const MomentumSet& p_src, double sigma);

struct HessianProducts {
  std::vector<Vec3> pq_alpha;
  std::vector<Vec3> pp_alpha;
  std::vector<Vec3> qq_beta;
  std::vector<Vec3> qp_beta;
};

HessianProducts hessian_products(const PointSet& q, const MomentumSet& p,
                                 const std::vector<Vec3>& alpha, const std::vector<Vec3>& beta,
                                 double sigma);

/// Arithmetic precision used by the free functions above (FP64 by default,
/// as the reference). Per thread.
void set_kernel_precision(Precision p);
Precision kernel_precision();

}  // namespace geoshoot
