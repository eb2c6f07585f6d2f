// epilogue.cu -- O(N) stage epilogues fused behind the O(N^2) sums.
//
// Forward: fold the S source-chunk partials in fixed order, form
//   dH/dp_i = 2 sum_j G_ij p_j,  dH/dq_i = -(2/s) sum_j (p_i.p_j) G_ij (q_i - q_j)
// (kernel_exact.hpp:46-52) and apply the integrator in place:
//   Euler  q += dt dH/dp, p -= dt dH/dq                      (shooting.cpp:110-114)
//   RK4    k_s = (dH/dp, -dH/dq); stage state y + w_s dt k_s; y += dt/6 (k1+2k2+2k3+k4)
//          with the sum accumulated left to right as in test_shooting.cpp:55-58.
// A non-finite result sets the 1-based step in *bad_step (atomicMin), the
// device equivalent of NonFiniteState(k + 1) (shooting.cpp:115).
// Backward: the adjoint update alpha += dt (pq - qq), beta += dt (pp - qp)
// (shooting.cpp:211-214).
#include "engine.h"
#define GS_TRACE_TU 3
#include "trace.cuh"

namespace gsb {

namespace {

template <typename R> struct Vec { R x, y, z; };

template <typename R>
__device__ __forceinline__ Vec<R> fold(const V4<R>* part, int S, int n_tgt, int per, int t,
                                       int which) {
  Vec<R> a{R(0), R(0), R(0)};
  for (int s = 0; s < S; ++s) {
    const V4<R> v = ld4(part + (size_t)per * ((size_t)s * n_tgt + t) + which);
    a.x += v.x; a.y += v.y; a.z += v.z;
  }
  return a;
}

__device__ __forceinline__ bool fin(double v) { return isfinite(v); }

template <int NT>
__device__ double block_sum(double v) {
  __shared__ double red[NT / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < NT / 32; ++w) s += red[w];
  return s;
}

constexpr int kEpiNT = 256;

template <typename R>
__global__ void __launch_bounds__(kEpiNT) k_fwd_epi(FwdEpi e) {
  GS_TRACE_HERE();
  const int t = blockIdx.x * kEpiNT + threadIdx.x;
  double edot = 0.0;
  if (t < e.n_tgt) {
    const int i = e.tgt_begin + t;
    const V4<R>* part = static_cast<const V4<R>*>(e.part);
    const Vec<R> A = fold<R>(part, e.S, e.n_tgt, e.parts_per_tgt, t, 0);
    const Vec<R> B = fold<R>(part, e.S, e.n_tgt, e.parts_per_tgt, t, 1);
    const R cp = R(e.cp), cq = R(e.cq);
    const R gpx = cp * A.x, gpy = cp * A.y, gpz = cp * A.z;  // dH/dp
    const R gqx = cq * B.x, gqy = cq * B.y, gqz = cq * B.z;  // dH/dq
    V4<R>* rec = static_cast<V4<R>*>(e.rec);
    if (e.dhdp_out) {
      e.dhdp_out[3 * t] = gpx; e.dhdp_out[3 * t + 1] = gpy; e.dhdp_out[3 * t + 2] = gpz;
    }
    if (e.dhdq_out) {
      e.dhdq_out[3 * t] = gqx; e.dhdq_out[3 * t + 1] = gqy; e.dhdq_out[3 * t + 2] = gqz;
    }
    if (e.energy_part) {
      const V4<R> p = ld4(rec + 2 * i + 1);
      edot = (double)p.x * (double)gpx + (double)p.y * (double)gpy + (double)p.z * (double)gpz;
    }
    if (e.update) {
      const R dt = R(e.dt);
      bool check = true;
      V4<R> q, p;
      if (e.integrator == GS_EULER) {
        q = ld4(rec + 2 * i);
        p = ld4(rec + 2 * i + 1);
        q.x += dt * gpx; q.y += dt * gpy; q.z += dt * gpz;
        p.x -= dt * gqx; p.y -= dt * gqy; p.z -= dt * gqz;
      } else {
        V4<R>* y = static_cast<V4<R>*>(e.y);
        V4<R>* ks = static_cast<V4<R>*>(e.ks);
        V4<R> yq, yp;
        if (e.stage == 0) {  // stage-0 records are the step-start state
          yq = ld4(rec + 2 * i);
          yp = ld4(rec + 2 * i + 1);
          st4(y + 2 * i, yq);
          st4(y + 2 * i + 1, yp);
        } else {
          yq = ld4(y + 2 * i);
          yp = ld4(y + 2 * i + 1);
        }
        // k = (dH/dp, -dH/dq); ks = k1 (+ 2 k2 + 2 k3 + k4)
        V4<R> kq = mk4<R>(gpx, gpy, gpz), kp = mk4<R>(-gqx, -gqy, -gqz);
        V4<R> sq, sp;
        if (e.stage == 0) {
          sq = kq; sp = kp;
        } else {
          const R w = e.stage == 3 ? R(1) : R(2);
          sq = ld4(ks + 2 * i); sp = ld4(ks + 2 * i + 1);
          sq.x += w * kq.x; sq.y += w * kq.y; sq.z += w * kq.z;
          sp.x += w * kp.x; sp.y += w * kp.y; sp.z += w * kp.z;
        }
        if (e.stage < 3) {
          st4(ks + 2 * i, sq);
          st4(ks + 2 * i + 1, sp);
          const R hw = (e.stage == 2 ? R(1) : R(0.5)) * dt;
          q = mk4<R>(yq.x + hw * kq.x, yq.y + hw * kq.y, yq.z + hw * kq.z);
          p = mk4<R>(yp.x + hw * kp.x, yp.y + hw * kp.y, yp.z + hw * kp.z);
          check = false;
        } else {
          const R h6 = dt / R(6);
          q = mk4<R>(yq.x + h6 * sq.x, yq.y + h6 * sq.y, yq.z + h6 * sq.z);
          p = mk4<R>(yp.x + h6 * sp.x, yp.y + h6 * sp.y, yp.z + h6 * sp.z);
        }
      }
      q.w = R(0); p.w = R(0);
      V4<R>* out = e.rec_out ? static_cast<V4<R>*>(e.rec_out) : rec;
      st4(out + 2 * i, q);
      st4(out + 2 * i + 1, p);
      for (int k = 0; k < e.peers.n; ++k) {  // fused all-gather: the peers' copies of slot i
        V4<R>* o = static_cast<V4<R>*>(e.peers.buf[k]);
        st4(o + 2 * i, q);
        st4(o + 2 * i + 1, p);
      }
      if (check && e.bad_step &&
          !(fin(q.x) && fin(q.y) && fin(q.z) && fin(p.x) && fin(p.y) && fin(p.z)))
        atomicMin(e.bad_step, e.step_dev ? *e.step_dev + 1 : e.step);
    }
  }
  if (e.energy_part) {
    const double s = block_sum<kEpiNT>(edot);
    if (threadIdx.x == 0) e.energy_part[blockIdx.x] = s;
  }
  if (e.step_inc) {  // (every block's read of *step_dev precedes its arrival)
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      unsigned* arrivals = reinterpret_cast<unsigned*>(e.step_inc) + 1;
      if (atomicAdd(arrivals, 1u) == gridDim.x - 1) {
        e.step_inc[0] += 1;
        *arrivals = 0;
      }
    }
  }
}

template <typename R>
__global__ void __launch_bounds__(kEpiNT) k_bwd_epi(BwdEpi e) {
  GS_TRACE_HERE();
  const int t = blockIdx.x * kEpiNT + threadIdx.x;
  if (t >= e.n_tgt) return;
  const int i = e.tgt_begin + t;
  const V4<R>* part = static_cast<const V4<R>*>(e.part);
  const Vec<R> A0 = fold<R>(part, e.S, e.n_tgt, 4, t, 0);
  const Vec<R> A1 = fold<R>(part, e.S, e.n_tgt, 4, t, 1);
  const Vec<R> A2 = fold<R>(part, e.S, e.n_tgt, 4, t, 2);
  const Vec<R> A3 = fold<R>(part, e.S, e.n_tgt, 4, t, 3);
  const R cpq = R(e.cpq), cpp = R(e.cpp), cqq = R(e.cqq), cqp = R(e.cqp);
  const Vec<R> pq{cpq * A0.x, cpq * A0.y, cpq * A0.z};
  const Vec<R> pp{cpp * A1.x, cpp * A1.y, cpp * A1.z};
  const Vec<R> qq{cqq * A2.x, cqq * A2.y, cqq * A2.z};
  const Vec<R> qp{cqp * A3.x, cqp * A3.y, cqp * A3.z};
  const Vec<R>* outs[4] = {&pq, &pp, &qq, &qp};
  for (int c = 0; c < 4; ++c)
    if (e.out[c]) {
      e.out[c][3 * t] = outs[c]->x; e.out[c][3 * t + 1] = outs[c]->y; e.out[c][3 * t + 2] = outs[c]->z;
    }
  if (e.update) {
    V4<R>* adj = static_cast<V4<R>*>(e.adj);
    V4<R> a = ld4(adj + 2 * i), b = ld4(adj + 2 * i + 1);
    const R dt = R(e.dt);
    a.x += dt * (pq.x - qq.x); a.y += dt * (pq.y - qq.y); a.z += dt * (pq.z - qq.z);
    b.x += dt * (pp.x - qp.x); b.y += dt * (pp.y - qp.y); b.z += dt * (pp.z - qp.z);
    V4<R>* out = e.adj_out ? static_cast<V4<R>*>(e.adj_out) : adj;
    st4(out + 2 * i, a);
    st4(out + 2 * i + 1, b);
    for (int k = 0; k < e.peers.n; ++k) {
      V4<R>* o = static_cast<V4<R>*>(e.peers.buf[k]);
      st4(o + 2 * i, a);
      st4(o + 2 * i + 1, b);
    }
  }
}

template <typename R>
__global__ void __launch_bounds__(kEpiNT) k_vel_epi(VelEpi e) {
  GS_TRACE_HERE();
  const int t = blockIdx.x * kEpiNT + threadIdx.x;
  if (t >= e.m) return;
  const Vec<R> A = fold<R>(static_cast<const V4<R>*>(e.part), e.S, e.m, 1, t, 0);
  const R sc = R(e.scale);
  const R vx = sc * A.x, vy = sc * A.y, vz = sc * A.z;
  if (e.v_out) { e.v_out[3 * t] = vx; e.v_out[3 * t + 1] = vy; e.v_out[3 * t + 2] = vz; }
  if (e.update) {
    V4<R>* ev = static_cast<V4<R>*>(e.ev);
    V4<R> y = ld4(ev + 2 * t);
    const R dt = R(e.dt);
    y.x += dt * vx; y.y += dt * vy; y.z += dt * vz;
    st4(ev + 2 * t, y);
    if (e.bad_step && !(fin(y.x) && fin(y.y) && fin(y.z))) atomicMin(e.bad_step, e.step);
  }
}

template <typename R>
__global__ void k_pack(const double* q, const double* p, int64_t n, V4<R>* rec, int* bad) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = q[3 * i], b = q[3 * i + 1], c = q[3 * i + 2];
  double x = 0, y = 0, z = 0;
  if (p) { x = p[3 * i]; y = p[3 * i + 1]; z = p[3 * i + 2]; }
  if (bad && !(fin(a) && fin(b) && fin(c) && fin(x) && fin(y) && fin(z))) atomicExch(bad, 1);
  st4(rec + 2 * i, mk4<R>(R(a), R(b), R(c)));
  st4(rec + 2 * i + 1, mk4<R>(R(x), R(y), R(z)));
}

template <typename R>
__global__ void k_unpack(const V4<R>* rec, int64_t n, double* q, double* p) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const V4<R> a = ld4(rec + 2 * i), b = ld4(rec + 2 * i + 1);
  if (q) { q[3 * i] = a.x; q[3 * i + 1] = a.y; q[3 * i + 2] = a.z; }
  if (p) { p[3 * i] = b.x; p[3 * i + 1] = b.y; p[3 * i + 2] = b.z; }
}

template <typename R>
__global__ void k_grad(const V4<R>* adj, const double* dhdp0, int64_t n, double* grad) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const V4<R> b = ld4(adj + 2 * i + 1);
  // grad = beta_0 + dH/dp(q0, p0), shooting.cpp:234
  grad[3 * i] = (double)b.x + dhdp0[3 * i];
  grad[3 * i + 1] = (double)b.y + dhdp0[3 * i + 1];
  grad[3 * i + 2] = (double)b.z + dhdp0[3 * i + 2];
}

template <typename R>
__global__ void __launch_bounds__(kEpiNT) k_adj_init(const V4<R>* recT, const double* target,
                                                     double lambda, int64_t n, V4<R>* adj,
                                                     double* sse_part) {
  const int64_t i = blockIdx.x * (int64_t)kEpiNT + threadIdx.x;
  double sse = 0.0;
  if (i < n) {
    const V4<R> q = ld4(recT + 2 * i);
    const double dx = (double)q.x - target[3 * i], dy = (double)q.y - target[3 * i + 1],
                 dz = (double)q.z - target[3 * i + 2];
    sse = dx * dx + dy * dy + dz * dz;
    const double l2 = 2.0 * lambda;  // alpha_T = 2 lambda (q_T - target), shooting.cpp:161-166
    st4(adj + 2 * i, mk4<R>(R(l2 * dx), R(l2 * dy), R(l2 * dz)));
    st4(adj + 2 * i + 1, mk4<R>(R(0), R(0), R(0)));
  }
  const double s = block_sum<kEpiNT>(sse);
  if (threadIdx.x == 0 && sse_part) sse_part[blockIdx.x] = s;
}


__global__ void k_reduce(const double* part, int count, double* out) {
  // one warp, fixed order per lane then fixed tree: deterministic
  double s = 0.0;
  for (int i = threadIdx.x; i < count; i += 32) s += part[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) *out = s;
}

inline int blocks_for(int64_t n, int nt) { return (int)std::max<int64_t>(1, (n + nt - 1) / nt); }

// per-block sums of the .w lane of partial vec4 `which` ([S][n][per] layout, S = 1)
template <typename R>
__global__ void __launch_bounds__(kEpiNT) k_sum_w(const V4<R>* part, int n, int per, int which,
                                                  double* out) {
  const int t = blockIdx.x * kEpiNT + threadIdx.x;
  const double v = t < n ? (double)ld4(part + (size_t)per * t + which).w : 0.0;
  const double s = block_sum<kEpiNT>(v);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

}  // namespace

namespace {
template <typename R>
__global__ void k_permute_records(const V4<R>* in, const int* perm, int64_t n, V4<R>* out) {
  const int64_t t = blockIdx.x * (int64_t)kEpiNT + threadIdx.x;
  if (t >= n) return;
  const int i = perm[t];
  st4(out + 2 * t, ld4(in + 2 * i));
  st4(out + 2 * t + 1, ld4(in + 2 * i + 1));
}
__global__ void k_gather_rows3(const double* in, const int* perm, int64_t n, double* out) {
  const int64_t t = blockIdx.x * (int64_t)kEpiNT + threadIdx.x;
  if (t >= n) return;
  const int64_t i = perm[t];
  out[3 * t] = in[3 * i];
  out[3 * t + 1] = in[3 * i + 1];
  out[3 * t + 2] = in[3 * i + 2];
}
__global__ void k_scatter_rows3(const double* in, const int* perm, int64_t n, double* out) {
  const int64_t t = blockIdx.x * (int64_t)kEpiNT + threadIdx.x;
  if (t >= n) return;
  const int64_t i = perm[t];
  out[3 * i] = in[3 * t];
  out[3 * i + 1] = in[3 * t + 1];
  out[3 * i + 2] = in[3 * t + 2];
}
}  // namespace

int permute_records(int prec, const void* in, const int* perm, int64_t n, void* out, cudaStream_t st) {
  const int nb = blocks_for(n, kEpiNT);
  if (prec == kF32)
    k_permute_records<float><<<nb, kEpiNT, 0, st>>>((const float4*)in, perm, n, (float4*)out);
  else
    k_permute_records<double><<<nb, kEpiNT, 0, st>>>((const double4*)in, perm, n, (double4*)out);
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}

int gather_rows3(const double* in, const int* perm, int64_t n, double* out, cudaStream_t st) {
  k_gather_rows3<<<blocks_for(n, kEpiNT), kEpiNT, 0, st>>>(in, perm, n, out);
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}

int scatter_rows3(const double* in, const int* perm, int64_t n, double* out, cudaStream_t st) {
  k_scatter_rows3<<<blocks_for(n, kEpiNT), kEpiNT, 0, st>>>(in, perm, n, out);
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}

int sum_part_w(int prec, const void* part, int n, int per, int which, double* block_out,
               int* blocks, cudaStream_t st) {
  const int nb = blocks_for(n, kEpiNT);
  if (prec == kF32)
    k_sum_w<float><<<nb, kEpiNT, 0, st>>>(static_cast<const float4*>(part), n, per, which, block_out);
  else
    k_sum_w<double><<<nb, kEpiNT, 0, st>>>(static_cast<const double4*>(part), n, per, which, block_out);
  GS_CUDA_OK(cudaGetLastError());
  *blocks = nb;
  return GS_OK;
}

int fwd_epilogue(int prec, const FwdEpi& e, cudaStream_t st, int* blocks_out) {
  const int nb = blocks_for(e.n_tgt, kEpiNT);
  if (blocks_out) *blocks_out = nb;
  if (prec == kF32) k_fwd_epi<float><<<nb, kEpiNT, 0, st>>>(e);
  else k_fwd_epi<double><<<nb, kEpiNT, 0, st>>>(e);
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}

int bwd_epilogue(int prec, const BwdEpi& e, cudaStream_t st) {
  const int nb = blocks_for(e.n_tgt, kEpiNT);
  if (prec == kF32) k_bwd_epi<float><<<nb, kEpiNT, 0, st>>>(e);
  else k_bwd_epi<double><<<nb, kEpiNT, 0, st>>>(e);
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}

int vel_epilogue(int prec, const VelEpi& e, cudaStream_t st) {
  const int nb = blocks_for(e.m, kEpiNT);
  if (prec == kF32) k_vel_epi<float><<<nb, kEpiNT, 0, st>>>(e);
  else k_vel_epi<double><<<nb, kEpiNT, 0, st>>>(e);
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}

int pack_records(int prec, const double* q, const double* p, int64_t n, void* rec, int* bad,
                 cudaStream_t st) {
  const int nb = blocks_for(n, 256);
  if (prec == kF32) k_pack<float><<<nb, 256, 0, st>>>(q, p, n, (float4*)rec, bad);
  else k_pack<double><<<nb, 256, 0, st>>>(q, p, n, (double4*)rec, bad);
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}

int unpack_records(int prec, const void* rec, int64_t n, double* q, double* p, cudaStream_t st) {
  const int nb = blocks_for(n, 256);
  if (prec == kF32) k_unpack<float><<<nb, 256, 0, st>>>((const float4*)rec, n, q, p);
  else k_unpack<double><<<nb, 256, 0, st>>>((const double4*)rec, n, q, p);
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}

int gradient_finalize(int prec, const void* adj, const double* dhdp0, int64_t n, double* grad,
                      cudaStream_t st) {
  const int nb = blocks_for(n, 256);
  if (prec == kF32) k_grad<float><<<nb, 256, 0, st>>>((const float4*)adj, dhdp0, n, grad);
  else k_grad<double><<<nb, 256, 0, st>>>((const double4*)adj, dhdp0, n, grad);
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}

int adjoint_init(int prec, const void* rec_T, const double* target, double lambda, int64_t n,
                 void* adj, double* sse_part, int* blocks, cudaStream_t st) {
  const int nb = blocks_for(n, kEpiNT);
  if (blocks) *blocks = nb;
  if (prec == kF32)
    k_adj_init<float><<<nb, kEpiNT, 0, st>>>((const float4*)rec_T, target, lambda, n, (float4*)adj, sse_part);
  else
    k_adj_init<double><<<nb, kEpiNT, 0, st>>>((const double4*)rec_T, target, lambda, n, (double4*)adj, sse_part);
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}


int reduce_sum(const double* part, int count, double* out, cudaStream_t st) {
  k_reduce<<<1, 32, 0, st>>>(part, count, out);
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}

int trace_install_epi(unsigned long long* buf) {
  GS_CUDA_OK(trace_install_here(buf));
  return GS_OK;
}

}  // namespace gsb
