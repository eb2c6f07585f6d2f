// microbench.cu -- measured FP32 / SFU / FP64 issue peaks of the device, the
// denominators of the all-pairs roofline (MEASURED_PEAKS.json only carries HBM
// and bf16 tensor numbers). Each thread runs 8 independent dependency chains,
// enough ILP to saturate the pipe; the grid fills every SM.
#include "engine.h"

namespace gsb {
namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) k_ffma(float* out, int iters, float a, float b) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) x[c] = fmaf(x[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

// all-register operands (FFMA R, R, R, R), the form the pair kernel issues
__global__ void __launch_bounds__(256) k_ffma_reg(float* out, int iters, const float* ab) {
  float x[kChains], a[kChains], b[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    x[c] = threadIdx.x * 1e-3f + c;
    a[c] = ab[c] + threadIdx.x * 1e-9f;
    b[c] = ab[8 + c];
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) x[c] = fmaf(x[c], a[(c + u) & 7], b[(c + 3 * u) & 7]);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

// packed FP32x2 FMA (FFMA2): counts 2 lane-FMAs per lane per instruction
__global__ void __launch_bounds__(256) k_ffma2(float* out, int iters, float a, float b) {
  unsigned long long x[kChains], av, bv;
  asm("mov.b64 %0, {%1, %1};" : "=l"(av) : "f"(a));
  asm("mov.b64 %0, {%1, %1};" : "=l"(bv) : "f"(b));
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    const float lo = threadIdx.x * 1e-3f + c, hi = lo + 0.5f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x[c]) : "f"(lo), "f"(hi));
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c)
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(av), "l"(bv));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[c]));
    s += lo + hi;
  }
  if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_ex2(float* out, int iters) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = -(threadIdx.x * 1e-4f + c * 1e-2f);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) x[c] = -ex2(x[c]);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5) out[threadIdx.x] = s;
}

}  // namespace
}  // namespace gsb

using namespace gsb;

extern "C" gs_status gs_microbench(int device, int32_t kind, double* ops_per_s) {
  if (!ops_per_s) return GS_INVALID_ARGUMENT;
  if (cudaSetDevice(device) != cudaSuccess) return GS_NO_DEVICE;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  const int blocks = prop.multiProcessorCount * 8, threads = 256;
  const int iters = kind == 2 ? 256 : 2048;
  void* out = nullptr;
  GS_CUDA_OK(cudaMalloc(&out, 4096));
  GS_CUDA_OK(cudaMemset(out, 0, 4096));
  if (kind == 3) {
    float ab[16];
    for (int c = 0; c < 16; ++c) ab[c] = c < 8 ? 0.9999f + 1e-6f * c : 1e-7f * c;
    GS_CUDA_OK(cudaMemcpy(out, ab, sizeof ab, cudaMemcpyHostToDevice));
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    if (kind == 0) k_ffma<<<blocks, threads>>>((float*)out, iters, 0.999999f, 1e-7f);
    else if (kind == 1) k_ex2<<<blocks, threads>>>((float*)out, iters);
    else if (kind == 3) k_ffma_reg<<<blocks, threads>>>((float*)out + 64, iters, (const float*)out);
    else if (kind == 4) k_ffma2<<<blocks, threads>>>((float*)out, iters, 0.999999f, 1e-7f);
    else k_dfma<<<blocks, threads>>>((double*)out, iters, 0.999999, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0) best = std::min(best, ms);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  GS_CUDA_OK(cudaGetLastError());
  // lane-operations per second (one FFMA / MUFU / DFMA per lane per op)
  const double ops = (double)blocks * threads * iters * 16.0 * kChains * (kind == 4 ? 2.0 : 1.0);
  *ops_per_s = ops / (best * 1e-3);
  return GS_OK;
}
