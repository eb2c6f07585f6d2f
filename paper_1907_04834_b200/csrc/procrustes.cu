// procrustes.cu -- rigid pre-alignment (reference
// procrustes.cpp:7-58): least-squares rotation + translation taking source
// onto target under index correspondence, reflection-corrected.
//
// The O(N) parts run on the device in FP64 with fixed-order reductions
// (deterministic): the two centroids, the 3x3 cross-covariance
// H = sum (s_i - s_mean)(t_i - t_mean)^T and the final transform of every
// point. The 3x3 SVD of H is host arithmetic on nine numbers (one-sided
// Jacobi; the reference uses Eigen's JacobiSVD, absent here).
#include <cmath>
#include <utility>

#include "engine.h"

#define GS_TRY_INT_AS(expr)                      \
  do {                                           \
    const int s__ = (expr);                      \
    if (s__ != GS_OK) return (gs_status)s__;     \
  } while (0)

namespace gsb {
namespace {

constexpr int kPNT = 256;

template <int K>
__device__ void block_sum_k(double (&v)[K], double* out) {
  __shared__ double red[K][kPNT / 32];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double x = v[k];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = x;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double s = 0.0;
    for (int w = 0; w < kPNT / 32; ++w) s += red[threadIdx.x][w];
    out[K * blockIdx.x + threadIdx.x] = s;
  }
}

// pass 0: sums of s and t (6); pass 1: cross-covariance about the means (9)
__global__ void __launch_bounds__(kPNT) k_moments(const double* s, const double* t, int64_t n,
                                                  const double* means, double* part) {
  if (!means) {
    double v[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t i = blockIdx.x * (int64_t)kPNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kPNT)
      for (int a = 0; a < 3; ++a) {
        v[a] += s[3 * i + a];
        v[3 + a] += t[3 * i + a];
      }
    block_sum_k<6>(v, part);
  } else {
    double v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t i = blockIdx.x * (int64_t)kPNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kPNT) {
      double ds[3], dt[3];
      for (int a = 0; a < 3; ++a) {
        ds[a] = s[3 * i + a] - means[a];
        dt[a] = t[3 * i + a] - means[3 + a];
      }
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) v[3 * r + c] += ds[r] * dt[c];
    }
    block_sum_k<9>(v, part);
  }
}

__global__ void k_fold(const double* part, int nb, int k, double* out, double scale) {
  const int c = threadIdx.x;
  if (c >= k) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[k * b + c];
  out[c] = s * scale;
}

__global__ void k_apply(const double* s, int64_t n, const double* tf, double* y) {
  const int64_t i = blockIdx.x * (int64_t)kPNT + threadIdx.x;
  if (i >= n) return;
  const double x0 = s[3 * i], x1 = s[3 * i + 1], x2 = s[3 * i + 2];
  for (int r = 0; r < 3; ++r)  // RigidTransform::apply, pipeline.hpp:16-20
    y[3 * i + r] = (tf[3 * r] * x0 + tf[3 * r + 1] * x1 + tf[3 * r + 2] * x2) + tf[9 + r];
}

// one-sided Jacobi SVD of a 3x3 matrix: A = U diag(sv) V^T, sv descending
void svd3(const double A[9], double U[9], double sv[3], double V[9]) {
  double a[9];
  for (int k = 0; k < 9; ++k) a[k] = A[k];
  for (int k = 0; k < 9; ++k) V[k] = (k % 4 == 0) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double al = 0, be = 0, ga = 0;
        for (int r = 0; r < 3; ++r) {
          al += a[3 * r + p] * a[3 * r + p];
          be += a[3 * r + q] * a[3 * r + q];
          ga += a[3 * r + p] * a[3 * r + q];
        }
        if (std::abs(ga) <= 1e-300) continue;
        off = std::max(off, std::abs(ga) / std::sqrt(al * be));
        const double zeta = (be - al) / (2.0 * ga);
        const double tn = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + tn * tn), s = c * tn;
        for (int r = 0; r < 3; ++r) {
          const double ap = a[3 * r + p], aq = a[3 * r + q];
          a[3 * r + p] = c * ap - s * aq;
          a[3 * r + q] = s * ap + c * aq;
          const double vp = V[3 * r + p], vq = V[3 * r + q];
          V[3 * r + p] = c * vp - s * vq;
          V[3 * r + q] = s * vp + c * vq;
        }
      }
    if (off < 1e-15) break;
  }
  int order[3] = {0, 1, 2};
  double nrm[3];
  for (int c = 0; c < 3; ++c)
    nrm[c] = std::sqrt(a[c] * a[c] + a[3 + c] * a[3 + c] + a[6 + c] * a[6 + c]);
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (nrm[order[j]] > nrm[order[i]]) std::swap(order[i], order[j]);
  double Vs[9], Us[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int c = 0; c < 3; ++c) {
    const int o = order[c];
    sv[c] = nrm[o];
    for (int r = 0; r < 3; ++r) {
      Vs[3 * r + c] = V[3 * r + o];
      if (nrm[o] > 0) Us[3 * r + c] = a[3 * r + o] / nrm[o];
    }
  }
  // complete U where singular values vanish (orthonormal completion)
  auto col = [&](int c, double* v) { for (int r = 0; r < 3; ++r) v[r] = Us[3 * r + c]; };
  auto set = [&](int c, const double* v) { for (int r = 0; r < 3; ++r) Us[3 * r + c] = v[r]; };
  if (!(sv[1] > 0)) {  // only u0 known: pick any unit vector orthogonal to it
    double u0[3];
    col(0, u0);
    double e[3] = {std::abs(u0[0]) < 0.9 ? 1.0 : 0.0, std::abs(u0[0]) < 0.9 ? 0.0 : 1.0, 0.0};
    const double d = e[0] * u0[0] + e[1] * u0[1] + e[2] * u0[2];
    double u1[3] = {e[0] - d * u0[0], e[1] - d * u0[1], e[2] - d * u0[2]};
    const double l = std::sqrt(u1[0] * u1[0] + u1[1] * u1[1] + u1[2] * u1[2]);
    for (double& x : u1) x /= l;
    set(1, u1);
  }
  if (!(sv[2] > 0)) {
    double u0[3], u1[3];
    col(0, u0);
    col(1, u1);
    const double u2[3] = {u0[1] * u1[2] - u0[2] * u1[1], u0[2] * u1[0] - u0[0] * u1[2],
                          u0[0] * u1[1] - u0[1] * u1[0]};
    set(2, u2);
  }
  for (int k = 0; k < 9; ++k) {
    U[k] = Us[k];
    V[k] = Vs[k];
  }
}

double det3(const double M[9]) {
  return M[0] * (M[4] * M[8] - M[5] * M[7]) - M[1] * (M[3] * M[8] - M[5] * M[6]) +
         M[2] * (M[3] * M[7] - M[4] * M[6]);
}

}  // namespace
}  // namespace gsb

using namespace gsb;

struct gs_ctx;  // the context only provides a device; the stream is local
extern "C" gs_status gs_procrustes_align(gs_ctx* ctx, int64_t n, const double* source,
                                         const double* target, double* rotation_rows,
                                         double* translation, double* aligned_out) {
  if (!ctx || !source || !target) return GS_INVALID_ARGUMENT;
  if (n < 3) {
    set_error("procrustes_align: needs at least 3 points");
    return GS_DEGENERATE;
  }
  cudaStream_t st;
  GS_CUDA_OK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct Guard {
    cudaStream_t s;
    DBuf a, b, y, part, m;
    ~Guard() { cudaStreamDestroy(s); }
  } g{st};
  const size_t bytes = sizeof(double) * 3 * n;
  const int nb = (int)std::min<int64_t>(296, (n + kPNT - 1) / kPNT);
  GS_TRY_INT_AS(g.a.ensure(bytes));
  GS_TRY_INT_AS(g.b.ensure(bytes));
  GS_TRY_INT_AS(g.y.ensure(bytes));
  GS_TRY_INT_AS(g.part.ensure(sizeof(double) * 9 * nb));
  GS_TRY_INT_AS(g.m.ensure(sizeof(double) * 32));
  GS_CUDA_OK(cudaMemcpyAsync(g.a.ptr, source, bytes, cudaMemcpyHostToDevice, st));
  GS_CUDA_OK(cudaMemcpyAsync(g.b.ptr, target, bytes, cudaMemcpyHostToDevice, st));
  double* means = g.m.as<double>();
  double* cov = means + 8;
  double* tf_dev = means + 20;
  k_moments<<<nb, kPNT, 0, st>>>(g.a.as<double>(), g.b.as<double>(), n, nullptr, g.part.as<double>());
  k_fold<<<1, 32, 0, st>>>(g.part.as<double>(), nb, 6, means, 1.0 / (double)n);
  k_moments<<<nb, kPNT, 0, st>>>(g.a.as<double>(), g.b.as<double>(), n, means, g.part.as<double>());
  k_fold<<<1, 32, 0, st>>>(g.part.as<double>(), nb, 9, cov, 1.0);
  double host[17];
  GS_CUDA_OK(cudaMemcpyAsync(host, means, sizeof(double) * 17, cudaMemcpyDeviceToHost, st));
  GS_CUDA_OK(cudaStreamSynchronize(st));
  const double* sm = host;
  const double* tm = host + 3;
  const double* H = host + 8;
  double U[9], sv[3], V[9];
  svd3(H, U, sv, V);
  if (!(sv[1] > 1e-12 * sv[0])) {  // collinear sources: rotation undetermined (:35-38)
    set_error("procrustes_align: rank-deficient cross-covariance (collinear points?)");
    return GS_DEGENERATE;
  }
  // R = V diag(1, 1, sign det(V U^T)) U^T
  double VUt[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      VUt[3 * r + c] = V[3 * r] * U[3 * c] + V[3 * r + 1] * U[3 * c + 1] + V[3 * r + 2] * U[3 * c + 2];
  const double d = det3(VUt) < 0.0 ? -1.0 : 1.0;
  double R[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      R[3 * r + c] = V[3 * r] * U[3 * c] + V[3 * r + 1] * U[3 * c + 1] + d * V[3 * r + 2] * U[3 * c + 2];
  double tf[12];
  for (int k = 0; k < 9; ++k) tf[k] = R[k];
  for (int r = 0; r < 3; ++r)
    tf[9 + r] = tm[r] - (R[3 * r] * sm[0] + R[3 * r + 1] * sm[1] + R[3 * r + 2] * sm[2]);
  if (rotation_rows)
    for (int k = 0; k < 9; ++k) rotation_rows[k] = tf[k];
  if (translation)
    for (int r = 0; r < 3; ++r) translation[r] = tf[9 + r];
  if (aligned_out) {
    GS_CUDA_OK(cudaMemcpyAsync(tf_dev, tf, sizeof tf, cudaMemcpyHostToDevice, st));
    k_apply<<<(int)((n + kPNT - 1) / kPNT), kPNT, 0, st>>>(g.a.as<double>(), n, tf_dev, g.y.as<double>());
    GS_CUDA_OK(cudaMemcpyAsync(aligned_out, g.y.ptr, bytes, cudaMemcpyDeviceToHost, st));
    GS_CUDA_OK(cudaStreamSynchronize(st));
  }
  return GS_OK;
}
