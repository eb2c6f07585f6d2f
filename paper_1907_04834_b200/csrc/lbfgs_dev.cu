// lbfgs_dev.cu -- the registration optimizer with device-resident state
// (SURVEY.md §8f rank 1). The L-BFGS iterate p0, the gradient, the search
// direction, the trial points and the m history pairs (s, y) all live in HBM,
// as do q0 and the target (uploaded once per optimisation); every
// objective/gradient is one evaluate() straight from those device arrays
// (evaluate_resident: no per-evaluation uploads), and the two-loop recursion
// and line-search vector algebra are device kernels. Only the scalars that
// steer the search (objective values, slopes, curvature tests) come back to
// the host, so the control flow is the reference's, step for step
// (proj/src/optimizer.cpp: two-loop recursion :37-58, strong-Wolfe search
// :82-189, minimize :215-299; restated on host vectors in optimizer.cpp).
//
// Reductions (dot products, max |.|) use a fixed two-level order: block
// partial sums over a fixed grid, then one block summing the partials in
// order -- deterministic, and equal to the host's sequential sums to
// rounding.
#include <chrono>
#include <cmath>
#include <limits>
#include <vector>

#include "engine.h"
#include "lbfgs.h"

namespace gsb {

namespace {

constexpr int kRedBlocks = 296, kRedNT = 256;
constexpr double kInf = std::numeric_limits<double>::infinity();

template <int NT>
__device__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < NT / 32; ++w) s += sh[w];
  __syncthreads();
  return s;
}

// part[b] = sum over the block's grid-stride share of a[i] * b[i] (or |a[i]| max)
__global__ void __launch_bounds__(kRedNT) k_dot_part(const double* a, const double* b, int64_t n,
                                                     double* part) {
  __shared__ double sh[kRedNT / 32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kRedNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRedNT)
    s += a[i] * b[i];
  s = block_sum<kRedNT>(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kRedNT) k_maxabs_part(const double* a, int64_t n, double* part) {
  __shared__ double sh[kRedNT / 32];
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kRedNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRedNT)
    m = fmax(m, fabs(a[i]));  // fmax drops NaN, like the host's std::max fold
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < kRedNT / 32; ++w) r = fmax(r, sh[w]);
    part[blockIdx.x] = r;
  }
}

// out[0] = scale * sum(part[0..nb)) in order; optional out[0] = 1 / that (rho)
__global__ void k_sum_fin(const double* part, int nb, const double* scale, int invert, double* out) {
  __shared__ double sh[kRedNT / 32];
  double s = 0.0;
  for (int k = threadIdx.x; k < nb; k += kRedNT) s += part[k];
  s = block_sum<kRedNT>(s, sh);
  if (threadIdx.x == 0) {
    if (scale) s *= *scale;
    *out = invert ? 1.0 / s : s;
  }
}

__global__ void k_max_fin(const double* part, int nb, double* out) {
  if (threadIdx.x != 0) return;
  double m = 0.0;
  for (int k = 0; k < nb; ++k) m = fmax(m, part[k]);
  *out = m;
}

// y += c * x, c = sign * (*coef) (device scalar) or a host value
__global__ void k_axpy(double* y, const double* x, int64_t n, double c, const double* coef,
                       const double* coef2) {
  double a = c;
  if (coef) a *= *coef;
  if (coef2) a = *coef - *coef2;  // (alpha_i - beta)
  for (int64_t i = blockIdx.x * (int64_t)kRedNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRedNT)
    y[i] += a * x[i];
}

// y *= num / den (device scalars)
__global__ void k_scale_ratio(double* y, int64_t n, const double* num, const double* den) {
  const double g = *num / *den;
  for (int64_t i = blockIdx.x * (int64_t)kRedNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRedNT)
    y[i] *= g;
}

// out = x0 + a * d; out = a - b; out = -a
__global__ void k_lin(double* out, const double* x0, double a, const double* d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)kRedNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRedNT)
    out[i] = x0[i] + a * d[i];
}
__global__ void k_diff(double* out, const double* a, const double* b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)kRedNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRedNT)
    out[i] = a[i] - b[i];
}
__global__ void k_neg(double* out, const double* a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)kRedNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRedNT)
    out[i] = -a[i];
}

struct DevVecs {
  cudaStream_t st;
  int64_t n;  // 3 x points
  int grid;
  DBuf part, scal;  // reduction partials; device scalars
  double* hs = nullptr;  // pinned host scalars

  double* sc(int k) { return scal.as<double>() + k; }
  int err = GS_OK;
  void chk(cudaError_t e) {
    if (e != cudaSuccess && err == GS_OK) err = cuda_fail(e, "lbfgs_dev", __FILE__, __LINE__);
  }
  // device scalar k = dot(a, b) [* scale], or its inverse
  void dot_dev(const double* a, const double* b, int k, const double* scale = nullptr, int inv = 0) {
    k_dot_part<<<grid, kRedNT, 0, st>>>(a, b, n, part.as<double>());
    k_sum_fin<<<1, kRedNT, 0, st>>>(part.as<double>(), grid, scale, inv, sc(k));
  }
  double to_host(int k) {
    chk(cudaMemcpyAsync(hs, sc(k), sizeof(double), cudaMemcpyDeviceToHost, st));
    chk(cudaStreamSynchronize(st));
    return *hs;
  }
  double dot(const double* a, const double* b) {
    dot_dev(a, b, 0);
    return to_host(0);
  }
  // max |a_i| ignoring NaN (as the host's std::max fold does)
  double max_abs(const double* a) {
    k_maxabs_part<<<grid, kRedNT, 0, st>>>(a, n, part.as<double>());
    k_max_fin<<<1, 32, 0, st>>>(part.as<double>(), grid, sc(0));
    return to_host(0);
  }
  void axpy(double* y, const double* x, double c, const double* coef = nullptr,
            const double* coef2 = nullptr) {
    k_axpy<<<grid, kRedNT, 0, st>>>(y, x, n, c, coef, coef2);
  }
  void lin(double* out, const double* x0, double a, const double* d) {
    k_lin<<<grid, kRedNT, 0, st>>>(out, x0, a, d, n);
  }
  void diff(double* out, const double* a, const double* b) { k_diff<<<grid, kRedNT, 0, st>>>(out, a, b, n); }
  void neg(double* out, const double* a) { k_neg<<<grid, kRedNT, 0, st>>>(out, a, n); }
  void copy(double* out, const double* a) {
    chk(cudaMemcpyAsync(out, a, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  }
};

// device scalars: 0..1 scratch, 2.. : rho[m], alpha[m], beta, gamma num/den
constexpr int kScRho = 8;

}  // namespace

// minimize() (optimizer.cpp:215-299) over device vectors; objective(x_dev,
// g_dev) -> f (+inf: rejected point). Returns the iterate in x_out (host).
int lbfgs_minimize_device(const std::function<double(const double*, double*)>& objective,
                          int64_t n3, const gs_opt_config& oc, cudaStream_t st,
                          const std::function<void(int, double, double, double)>& on_iterate,
                          double* x_out, LbfgsResult& res) {
  const auto t0 = std::chrono::steady_clock::now();
  auto ms = [&] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  };
  const int m = std::max(1, oc.memory);
  DevVecs V;
  V.st = st;
  V.n = n3;
  V.grid = (int)std::min<int64_t>(kRedBlocks, std::max<int64_t>(1, (n3 + kRedNT - 1) / kRedNT));
  GS_TRY_INT(V.part.ensure(sizeof(double) * kRedBlocks));
  GS_TRY_INT(V.scal.ensure(sizeof(double) * (kScRho + 2 * (m + 1) + 8)));
  GS_CUDA_OK(cudaMallocHost(&V.hs, 4 * sizeof(double)));
  struct Pinned {
    double* p;
    ~Pinned() { cudaFreeHost(p); }
  } pin{V.hs};
  double* rho = V.sc(kScRho);          // [m + 1] ring slots
  double* alpha = rho + (m + 1);       // [m + 1]
  double* beta = alpha + (m + 1);      // scratch
  double* gnum = beta + 1;
  double* gden = beta + 2;
  // vectors: x, g, d, trial x / g, best point, m + 1 history slots (s, y)
  const size_t vb = sizeof(double) * (size_t)n3;
  std::vector<DBuf> bufs(7 + 2 * (m + 1));
  for (DBuf& b : bufs) GS_TRY_INT(b.ensure(vb));
  double* x = bufs[0].as<double>();
  double* g = bufs[1].as<double>();
  double* d = bufs[2].as<double>();
  double* xt = bufs[3].as<double>();
  double* gt = bufs[4].as<double>();
  std::vector<double*> S(m + 1), Y(m + 1);
  for (int k = 0; k <= m; ++k) {
    S[k] = bufs[7 + 2 * k].as<double>();
    Y[k] = bufs[8 + 2 * k].as<double>();
  }
  std::vector<int> hist;  // ring slots, oldest first
  int evaluations = 0;
  auto F = [&](const double* xv, double* gv) {
    ++evaluations;
    return objective(xv, gv);
  };

  GS_CUDA_OK(cudaMemsetAsync(x, 0, vb, st));
  res.f = F(x, g);
  if (!std::isfinite(res.f)) throw NonFiniteStart{};
  res.grad_inf = V.max_abs(g);
  if (on_iterate) on_iterate(0, res.f, res.grad_inf, ms());
  res.reason = -1;
  res.iterations = 0;
  for (int it = 1; it <= oc.max_iterations; ++it) {
    if (res.grad_inf <= oc.gradient_tolerance) {
      res.reason = GS_TERM_GRADIENT_TOLERANCE;
      break;
    }
    // direction: d = -H g by the two-loop recursion, scalars kept on the device
    V.copy(d, g);
    if (!hist.empty()) {
      for (int i = (int)hist.size(); i-- > 0;) {
        const int k = hist[i];
        V.dot_dev(S[k], d, kScRho + (m + 1) + k, rho + k);  // alpha_k = rho_k s_k.d
        V.axpy(d, Y[k], -1.0, alpha + k);
      }
      const int last = hist.back();
      V.dot_dev(S[last], Y[last], kScRho + 2 * (m + 1) + 1);  // gamma = s.y / y.y
      V.dot_dev(Y[last], Y[last], kScRho + 2 * (m + 1) + 2);
      k_scale_ratio<<<V.grid, kRedNT, 0, st>>>(d, n3, gnum, gden);
      for (int i = 0; i < (int)hist.size(); ++i) {
        const int k = hist[i];
        V.dot_dev(Y[k], d, kScRho + 2 * (m + 1), rho + k);  // beta = rho_k y_k.d
        V.axpy(d, S[k], 1.0, alpha + k, beta);               // d += (alpha_k - beta) s_k
      }
    }
    V.neg(d, d);
    double gd = V.dot(g, d);
    if (gd >= 0.0) {  // stale curvature: restart from steepest descent
      hist.clear();
      V.neg(d, g);
      gd = V.dot(g, d);
    }
    const double a0 = hist.empty() ? 1.0 / std::max(1.0, res.grad_inf) : 1.0;
    // strong-Wolfe line search (optimizer.cpp:82-189); slope0 = g.d
    const double slope0 = gd;
    bool ok = false;
    double f_new = kInf;
    if (slope0 < 0.0) {
      auto decreases = [&](double a, double fa) { return fa <= res.f + oc.sufficient_decrease * a * slope0; };
      auto curvature_ok = [&](double slope) { return std::abs(slope) <= -oc.curvature * slope0; };
      int trials = 0;
      double best_a = 0.0, best_f = res.f;
      double a_prev = 0.0, f_prev = res.f, a = a0;
      double lo = -1.0, hi = -1.0, f_lo = 0.0;
      bool bracketed = false;
      while (trials < oc.max_trials) {
        const double at = bracketed ? 0.5 * (lo + hi) : a;
        V.lin(xt, x, at, d);
        const double fa = F(xt, gt);
        ++trials;
        const double slope = std::isfinite(fa) ? V.dot(gt, d) : 0.0;
        if (!bracketed) {
          if (!std::isfinite(fa) || !decreases(at, fa) || (trials > 1 && fa >= f_prev)) {
            lo = a_prev;
            f_lo = f_prev;
            hi = at;
            bracketed = true;
            continue;
          }
        } else if (!std::isfinite(fa) || !decreases(at, fa) || fa >= f_lo) {
          hi = at;
          continue;
        }
        if (fa < best_f) {
          best_a = at;
          best_f = fa;
        }
        if (curvature_ok(slope)) {
          ok = true;
          f_new = fa;
          break;
        }
        if (!bracketed) {
          if (slope >= 0.0) {
            lo = at;
            f_lo = fa;
            hi = a_prev;
            bracketed = true;
            continue;
          }
          a_prev = at;
          f_prev = fa;
          a = 2.0 * at;
        } else {
          if (slope * (hi - lo) >= 0.0) hi = lo;
          lo = at;
          f_lo = fa;
        }
      }
      if (!ok && best_a > 0.0 && best_f < res.f) {  // budget spent: the best decrease point
        V.lin(xt, x, best_a, d);
        const double fb = F(xt, gt);
        if (std::isfinite(fb) && fb < res.f) {
          ok = true;
          f_new = fb;
        }
      }
    }
    GS_TRY_INT(V.err);
    if (!ok) {
      res.reason = GS_TERM_LINE_SEARCH_FAILURE;
      break;
    }
    const double gt_inf = V.max_abs(gt);
    if (!std::isfinite(gt_inf)) {
      res.reason = GS_TERM_NON_FINITE;
      break;
    }
    // history pair (s, y) into a free ring slot, curvature-gated (:271-277)
    int slot = 0;
    {
      std::vector<bool> used(m + 1, false);
      for (int k : hist) used[k] = true;
      while (used[slot]) ++slot;
    }
    V.diff(S[slot], xt, x);
    V.diff(Y[slot], gt, g);
    const double sy = V.dot(S[slot], Y[slot]);
    const double ss = V.dot(S[slot], S[slot]);
    const double yy = V.dot(Y[slot], Y[slot]);
    if (sy > 1e-10 * std::sqrt(ss) * std::sqrt(yy)) {
      V.dot_dev(S[slot], Y[slot], kScRho + slot, nullptr, 1);  // rho = 1 / s.y
      hist.push_back(slot);
      if ((int)hist.size() > oc.memory) hist.erase(hist.begin());
    }
    const double f_prev = res.f;
    std::swap(x, xt);
    std::swap(g, gt);
    res.f = f_new;
    res.grad_inf = gt_inf;
    res.iterations = it;
    if (on_iterate) on_iterate(it, res.f, res.grad_inf, ms());
    GS_TRY_INT(V.err);
    if (std::abs(f_prev - res.f) <= oc.relative_objective_tolerance * std::max(1.0, std::abs(res.f))) {
      res.reason = GS_TERM_OBJECTIVE_TOLERANCE;
      break;
    }
  }
  if (res.reason < 0)
    res.reason = res.grad_inf <= oc.gradient_tolerance ? GS_TERM_GRADIENT_TOLERANCE
                                                       : GS_TERM_MAX_ITERATIONS;
  res.evaluations = evaluations;
  GS_CUDA_OK(cudaMemcpyAsync(x_out, x, vb, cudaMemcpyDeviceToHost, st));
  GS_CUDA_OK(cudaStreamSynchronize(st));
  return V.err;
}

}  // namespace gsb
