// gs_common.cuh -- shared device types and helpers for the sm_100a kernels.
//
// Layout in HBM: every point is a record of two 4-vectors
// {q.x, q.y, q.z, 0 | p.x, p.y, p.z, 0} in the working precision (32 B in
// FP32, 64 B in FP64). Records are the integrator state, the all-pairs source
// tiles and the unit of the multi-GPU all-gather. The pad lane keeps every
// load a single 16-B (FP32) or two 16-B (FP64) vector transaction.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace gsb {

constexpr double kLog2e = 1.4426950408889634073599246810019;

template <typename R> struct V4T;
template <> struct V4T<float> { using type = float4; };
template <> struct V4T<double> { using type = double4; };
template <typename R> using V4 = typename V4T<R>::type;

template <typename R>
__host__ __device__ inline V4<R> mk4(R x, R y, R z, R w = R(0)) {
  V4<R> v; v.x = x; v.y = y; v.z = z; v.w = w; return v;
}

// Loads a 4-vector as 16-B vector transactions (double4 = 2 x 16 B).
__device__ __forceinline__ float4 ld4(const float4* p) { return *p; }
__device__ __forceinline__ double4 ld4(const double4* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = q[0], b = q[1];
  return make_double4(a.x, a.y, b.x, b.y);
}
// Two consecutive 4-vectors (32 B, 32-B aligned) in one load: sm_100's 256-bit
// LDG (LDG.E.ENL2.256) for FP32 -- one LSU instruction and one sector per lane
// instead of two 128-bit loads; FP64 (64 B) stays at 16-B transactions.
__device__ __forceinline__ void ld8(const float4* p, float4& a, float4& b) {
  asm("ld.global.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(p));
}
__device__ __forceinline__ void ld8(const double4* p, double4& a, double4& b) {
  a = ld4(p);
  b = ld4(p + 1);
}
__device__ __forceinline__ void st4(float4* p, float4 v) { *p = v; }
__device__ __forceinline__ void st4(double4* p, double4 v) {
  double2* q = reinterpret_cast<double2*>(p);
  q[0] = make_double2(v.x, v.y);
  q[1] = make_double2(v.z, v.w);
}

// exp2 on the SFU: one MUFU.EX2, flush-to-zero (underflow -> 0 is exactly the
// behaviour wanted for far pairs).
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- packed FP32x2 arithmetic (sm_100 FFMA2 / FMUL2 / FADD2) ----
// Two targets share one 64-bit register pair; a source coordinate enters as a
// scalar operand broadcast to both halves, so one issue slot does the work of
// two scalar FP32 instructions.
struct f2 {
  unsigned long long v;
};
__device__ __forceinline__ f2 pk2(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void up2(f2 a, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a.v));
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return r;
}
__device__ __forceinline__ f2 bc2(float x) { return pk2(x, x); }
// 2^-x on the SFU for both halves (the negation folds into MUFU's operand)
__device__ __forceinline__ f2 nex2x2(f2 r2) {
  float lo, hi;
  up2(r2, lo, hi);
  return pk2(ex2(-lo), ex2(-hi));
}

// Per-call constants of the Gaussian kernel G(r) = exp(-r^2 / (2 sigma^2)).
// FP32 kernels work in pre-scaled coordinates x' = kappa (x - c0) with
// kappa^2 = log2(e) / (2 s), so that G = 2^(-|x'_i - x'_j|^2): one MUFU.EX2 per
// pair and no per-pair multiply. c0 (the centre of the
// initial bounding box) keeps |x'| small so the FP32 differences stay sharp.
// FP64 kernels use unscaled coordinates and the reference's own expression
// exp(-|d|^2 * inv_two_s) (kernel_exact.cpp:7-9).
struct KernelConsts {
  double sigma, s, inv_s, inv_two_s, two_over_s;
  double kappa;        // sqrt(log2e / (2 s))
  double c0[3];        // FP32 centring
  double ext[3];       // extent of the caller's point set (host bounding box; 0 = unknown):
                       // sizes the Barnes-Hut walk's node windows (bh.cu bh_tasks)
};

inline KernelConsts make_consts(double sigma, const double* c0) {
  KernelConsts k;
  k.sigma = sigma;
  k.s = sigma * sigma;
  k.inv_s = 1.0 / k.s;
  k.inv_two_s = 1.0 / (2.0 * k.s);
  k.two_over_s = 2.0 / k.s;
  k.kappa = __builtin_sqrt(kLog2e / (2.0 * k.s));
  for (int a = 0; a < 3; ++a) k.c0[a] = c0 ? c0[a] : 0.0;
  for (int a = 0; a < 3; ++a) k.ext[a] = 0.0;
  return k;
}

// Converts to int or to gs_status so the macro works in both kinds of function.
struct StatusCode {
  int v;
  operator int() const { return v; }
  template <typename E, typename = typename std::enable_if<std::is_enum<E>::value>::type>
  operator E() const { return static_cast<E>(v); }
};

#define GS_CUDA_OK(expr)                                               \
  do {                                                                 \
    cudaError_t e__ = (expr);                                          \
    if (e__ != cudaSuccess)                                            \
      return ::gsb::StatusCode{::gsb::cuda_fail(e__, #expr, __FILE__, __LINE__)}; \
  } while (0)

}  // namespace gsb

// Programmatic dependent launch (PDL): kernels launched with pdl_launch()
// may be scheduled while their predecessor in the stream is still running;
// GS_PDL_ENTRY, the first statement of every such kernel, lets the NEXT
// kernel start launching (its CTAs then park at their own entry) and waits
// for the predecessor's completion and memory before touching its outputs.
// In a kernel launched normally both instructions are no-ops. Chains of short
// dependent kernels (the tree build) overlap each launch with the previous
// kernel's tail instead of paying it in full.
#ifndef GS_TRACE_HERE
#define GS_TRACE_HERE() ((void)0)  // trace.cuh: kernel start times (GS_TRACE tooling)
#endif
#define GS_PDL_ENTRY()                                         \
  do {                                                         \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
    asm volatile("griddepcontrol.wait;" ::: "memory");         \
    GS_TRACE_HERE();                                           \
  } while (0)

template <typename... P, typename... A>
inline cudaError_t pdl_launch(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<A&&>(args)...);
}
