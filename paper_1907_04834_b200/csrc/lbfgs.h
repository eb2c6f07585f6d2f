// lbfgs.h -- the generic L-BFGS / strong-Wolfe engine of optimizer.cpp
// (reference minimize(), optimizer.cpp:215-299), shared by gs_optimize (device
// evaluate() objective) and the C++ API's geoshoot::minimize.
#pragma once

#include <cstdint>
#include <functional>

#include <cuda_runtime.h>
#include <vector>

#include "geoshoot_b200.h"

namespace gsb {

using LbfgsObjective = std::function<double(const std::vector<double>& x, std::vector<double>& grad)>;
using LbfgsCallback = std::function<void(int iteration, double f, double grad_inf, double wall_ms)>;

struct LbfgsResult {
  std::vector<double> x;
  double f = 0.0;
  double grad_inf = 0.0;
  int reason = GS_TERM_MAX_ITERATIONS;  // gs_termination
  int iterations = 0;
  int evaluations = 0;
};

struct NonFiniteStart {};  // objective non-finite at x0 (NonFiniteObjectiveAtStart)

LbfgsResult lbfgs_minimize(const LbfgsObjective& objective, std::vector<double> x0,
                           const gs_opt_config& config, const LbfgsCallback& on_iterate = {});

// The same minimize() from x0 = 0 with every vector in HBM (lbfgs_dev.cu):
// objective(x_dev, g_dev) -> f (+inf: rejected); the final iterate goes to
// x_out (host, n3 doubles). Returns a gs_status.
int lbfgs_minimize_device(const std::function<double(const double*, double*)>& objective,
                          int64_t n3, const gs_opt_config& config, cudaStream_t stream,
                          const LbfgsCallback& on_iterate, double* x_out, LbfgsResult& result);

}  // namespace gsb
