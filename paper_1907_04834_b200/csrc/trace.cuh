// trace.cuh -- kernel start-time trace for measuring a captured (graph)
// step's composition on the device, where host-side events cannot look:
// with a buffer installed (gs_trace), thread 0 of block 0 of every traced
// kernel appends {tag, %globaltimer} at its start; consecutive starts give
// each kernel's share of the step (its run time + the launch gap after it).
// Tag = translation unit << 16 | source line of the trace point. Off (null
// buffer): one predicated-off branch in one thread per kernel.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef GS_TRACE_TU
#error "define GS_TRACE_TU (1 tree, 2 bh, 3 epilogue) before including trace.cuh"
#endif

static __device__ unsigned long long* gs_trace_buf = nullptr;  // [0] count, then {tag, t} pairs
constexpr int kTraceMax = 16384;

#undef GS_TRACE_HERE
#define GS_TRACE_HERE()                                                                   \
  do {                                                                                   \
    if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && gs_trace_buf) {        \
      unsigned long long t_;                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
      const unsigned long long k_ = atomicAdd(gs_trace_buf, 1ull);                       \
      if (k_ < (unsigned long long)kTraceMax) {                                          \
        gs_trace_buf[1 + 2 * k_] = ((unsigned long long)GS_TRACE_TU << 16) | __LINE__;   \
        gs_trace_buf[2 + 2 * k_] = t_;                                                   \
      }                                                                                  \
    }                                                                                    \
  } while (0)

static inline cudaError_t trace_install_here(unsigned long long* buf) {
  return cudaMemcpyToSymbol(gs_trace_buf, &buf, sizeof buf);
}
