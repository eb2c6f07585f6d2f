// engine.h -- internal interfaces between the C-ABI (capi.cu) and the kernels.
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "gs_common.cuh"
#include "geoshoot_b200.h"

namespace gsb {

enum { kF64 = GS_F64, kF32 = GS_F32 };

struct Device {
  int id = 0;
  int sms = 148;
};

#define GS_TRY_INT(expr)        \
  do {                          \
    const int s__ = (expr);     \
    if (s__ != GS_OK) return s__; \
  } while (0)

// Records the failing call in the thread's error slot; returns GS_CUDA_ERROR.
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);
void set_error(const std::string& msg);

// Growable device buffer (cudaMalloc, never shrinks).
// bumped on every device (re)allocation or free of a DBuf: cached CUDA graphs
// hold raw buffer pointers and re-validate them when it moved
extern std::atomic<unsigned long long> g_dbuf_epoch;

struct DBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  int ensure(size_t need);
  void release();
  template <typename T> T* as() const { return static_cast<T*>(ptr); }
  ~DBuf() { release(); }
};

// Optional event timing of the dominant kernels inside a flow (bench roofline):
// channel 0 = the O(N^2) / traversal kernel, channel 1 = the tree build,
// 2..5 = tree-build phases (bbox+keys, sort, topology, aggregates).
struct KTimer {
  static constexpr int kChannels = 8;
  std::vector<cudaEvent_t> ev[kChannels];
  std::vector<double> host_us[kChannels];  // GS_KT_VERBOSE: host clock at each mark
  size_t used[kChannels] = {0, 0, 0, 0, 0, 0, 0, 0};
  void mark(int ch, cudaStream_t st) {
    if (used[ch] == ev[ch].size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev[ch].push_back(e);
      host_us[ch].push_back(0.0);
    }
    host_us[ch][used[ch]] = (double)std::chrono::duration_cast<std::chrono::microseconds>(
        std::chrono::steady_clock::now().time_since_epoch()).count();
    cudaEventRecord(ev[ch][used[ch]++], st);
  }
  // sum of (end - start) over the recorded pairs; resets
  double drain(int ch, int64_t* pairs) {
    static const bool verbose = std::getenv("GS_KT_VERBOSE") != nullptr;
    double ms = 0.0;
    for (size_t k = 0; k + 1 < used[ch]; k += 2) {
      float v = 0.f;
      cudaEventSynchronize(ev[ch][k + 1]);
      cudaEventElapsedTime(&v, ev[ch][k], ev[ch][k + 1]);
      ms += v;
      if (verbose)
        std::fprintf(stderr, "[kt] ch %d pair %zu: %.3f ms (host %.3f ms, host t %.3f ms)\n", ch,
                     k / 2, v, (host_us[ch][k + 1] - host_us[ch][k]) / 1e3,
                     std::fmod(host_us[ch][k] / 1e3, 1e5));
    }
    if (pairs) *pairs = (int64_t)(used[ch] / 2);
    used[ch] = 0;
    return ms;
  }
  ~KTimer() {
    for (auto& v : ev)
      for (cudaEvent_t e : v) cudaEventDestroy(e);
  }
};
extern thread_local KTimer* g_ktimer;
inline void kt_mark(int ch, cudaStream_t st) {
  if (g_ktimer) g_ktimer->mark(ch, st);
}

// kernel start-time trace (trace.cuh): installs the buffer in each traced unit
int trace_install_tree(unsigned long long* buf);
int trace_install_bh(unsigned long long* buf);
int trace_install_epi(unsigned long long* buf);

inline size_t vec_bytes(int prec) { return prec == kF32 ? sizeof(float4) : sizeof(double4); }

// ---- exact RHS in Morton order with the FP32 underflow cutoff (allpairs.cu)
int rhs_sorted_partials(const Device& dev, const void* srec, const int* perm, int n,
                        void* part, int part_cap_chunks, DBuf& boxes, float cut2,
                        cudaStream_t st);

// ---- all-pairs (allpairs.cu); return the number of source chunks S used,
// ---- or -1 if S would exceed part_cap_chunks.
// plan_tgt > 0: launch n_tgt targets under the plan of a plan_tgt-target
// problem (kernel variant, targets per thread, source chunking), so a shard's
// partial sums are bit-identical to the plan_tgt-target run's (multi-device).
int rhs_partials(const Device& dev, int prec, const void* rec, int n, int tgt_begin, int n_tgt,
                 const KernelConsts& kc, void* part, int part_cap_chunks, cudaStream_t st,
                 int plan_tgt = -1);
// ---- symmetric exact FP32 RHS (allpairs.cu k_rhs_sym_f32x2): each unordered
// tile pair once, both ends fed; T = sym_tiles(n) partial slots per target.
void set_exact_pairs(int mode);
bool use_sym(int prec, int n, int tgt_begin, int n_tgt, int plan_tgt);
int sym_tiles(int n);
size_t sym_part_bytes(int n);
bool sym_grouped(int n);  // diagonal groups + running sum (slots over budget)
int sym_launches(int n);
int rhs_sym_partials(const void* rec, int n, const KernelConsts& kc, void* part, cudaStream_t st);
// multi-GPU rows of the symmetric RHS: this rank's tile-pair rows into part
// (T slots x n), folded per target into out (n x 2 float4); returns T
int rhs_sym_rows(const void* rec, int n, const KernelConsts& kc, void* part, void* out, int rank,
                 int world, cudaStream_t st);
// FP64 symmetric RHS (k_rhs_sym_f64, diagonal groups folded into a running
// sum): returns S = 1 (part holds the running sum first)
bool use_sym_f64(int n, int tgt_begin, int n_tgt, int plan_tgt);
size_t sym_f64_part_bytes(int n);
int rhs_sym_f64_partials(const void* rec, int n, const KernelConsts& kc, void* part,
                         cudaStream_t st);
int sym_f64_launches(int n);
int sym_f64_tiles(int n);
// bytes hess_partials needs in part for this problem (symmetric: T slots x 64 B)
size_t hess_part_bytes(int prec, int n, int tgt_begin, int n_tgt, int plan_tgt = -1);
int hess_partials(const Device& dev, int prec, const void* rec, const void* adj, int n,
                  int tgt_begin, int n_tgt, const KernelConsts& kc, void* part,
                  int part_cap_chunks, cudaStream_t st, int plan_tgt = -1);
int vel_partials(const Device& dev, int prec, const void* rec, int n, const void* ev, int m,
                 const KernelConsts& kc, void* part, int part_cap_chunks, cudaStream_t st);
constexpr int kMaxChunks = 16;

// ---- epilogues (epilogue.cu) -----------------------------------------------
// Multi-device flows (gs_create_multi): a stage epilogue stores each updated
// target record into its own buffer AND into the same slot of every peer's
// buffer (P2P stores over NVLink / NVSwitch), so the per-stage all-gather of
// the shards is fused into the epilogue -- no separate collective.
constexpr int kMaxPeers = 15;
struct PeerOut {
  void* buf[kMaxPeers] = {};
  int n = 0;
};
// Forward stage epilogue: folds partials A = sum g p, B = sum c d (per target),
// forms dH/dp = cp * A, dH/dq = cq * B and applies the integrator.
struct FwdEpi {
  int n_tgt = 0, tgt_begin = 0, S = 1, parts_per_tgt = 2;
  const void* part = nullptr;
  void* rec = nullptr;      // [n][2] records read for the targets
  void* rec_out = nullptr;  // where updated target records go (nullptr = rec, in place)
  void* y = nullptr;    // RK4: step-start records
  void* ks = nullptr;   // RK4: k1 + 2 k2 + 2 k3 (+ k4)
  int integrator = GS_EULER, stage = 0, update = 1;
  double dt = 0.0, cp = 2.0, cq = 0.0;
  double* dhdp_out = nullptr;  // optional double[3 n_tgt]
  double* dhdq_out = nullptr;
  double* energy_part = nullptr;  // optional per-block partial of <p, dH/dp>
  int* bad_step = nullptr;        // atomicMin on non-finite output
  int step = 0;                   // step index (1-based) reported on non-finite
  const int* step_dev = nullptr;  // if set: step = *step_dev + 1 (graph-replayable)
  int* step_inc = nullptr;  // a step's final stage: the last block to finish increments
                            // step_inc[0] (the step counter; step_inc[1]: arrivals)
  PeerOut peers;                  // multi-device: the updated records go here too
};
int fwd_epilogue(int prec, const FwdEpi& e, cudaStream_t st, int* blocks_out);

struct BwdEpi {
  int n_tgt = 0, tgt_begin = 0, S = 1;
  const void* part = nullptr;
  void* adj = nullptr;  // [n][2] (alpha, beta) updated in place when update != 0
  void* adj_out = nullptr;  // where the updated adjoints go (nullptr = adj, in place)
  PeerOut peers;            // multi-device: the updated adjoints go here too
  int update = 1;
  double dt = 0.0, cpq = 0.0, cpp = 2.0, cqq = 0.0, cqp = 0.0;
  double* out[4] = {nullptr, nullptr, nullptr, nullptr};  // pq, pp, qq, qp (optional)
};
int bwd_epilogue(int prec, const BwdEpi& e, cudaStream_t st);

// Velocity epilogue: v = scale * sum partials; either written out (double) or
// used to advect eval records y += dt * v in place.
struct VelEpi {
  int m = 0, S = 1;
  const void* part = nullptr;
  void* ev = nullptr;
  double scale = 1.0, dt = 0.0;
  int update = 0;
  double* v_out = nullptr;
  int* bad_step = nullptr;
  int step = 0;
};
int vel_epilogue(int prec, const VelEpi& e, cudaStream_t st);

// pack host-layout doubles [n][3] (device copy) into records; flags non-finite
int pack_records(int prec, const double* q, const double* p, int64_t n, void* rec, int* bad,
                 cudaStream_t st);
int unpack_records(int prec, const void* rec, int64_t n, double* q, double* p, cudaStream_t st);
// grad[i] = beta_i + dhdp0[i]
int gradient_finalize(int prec, const void* adj, const double* dhdp0, int64_t n, double* grad,
                      cudaStream_t st);
// alpha = 2 lambda (q_T - target), beta = 0
int adjoint_init(int prec, const void* rec_T, const double* target, double lambda, int64_t n,
                 void* adj, double* sse_part, int* blocks, cudaStream_t st);
int reduce_sum(const double* part, int count, double* out, cudaStream_t st);
// out[t] = in[perm[t]] (records, [n][2] V4) / out[perm[t]] = in[t] (double [n][3])
int permute_records(int prec, const void* in, const int* perm, int64_t n, void* out, cudaStream_t st);
int scatter_rows3(const double* in, const int* perm, int64_t n, double* out, cudaStream_t st);
// out[t] = in[perm[t]] (double [n][3])
int gather_rows3(const double* in, const int* perm, int64_t n, double* out, cudaStream_t st);
// per-block FP64 sums of the .w lane of partial vec4 `which` of n targets ([n][per] layout)
int sum_part_w(int prec, const void* part, int n, int per, int which, double* block_out,
               int* blocks, cudaStream_t st);
// ++*counter on the device (the step counter of graph-replayed flows)

}  // namespace gsb

struct gs_ctx;
namespace gsb {
// evaluate() with device-resident inputs (capi.cu): q0_dev / p0_dev /
// target_dev double [n][3]; box = {c0, ext} of q0's host bounding box; the
// gradient stays in grad_dev. Used by the device-resident optimizer.
int evaluate_resident(gs_ctx* c, const gs_config* cfg, int64_t n, const double* q0_dev,
                      const double* box, const double* p0_dev, const double* target_dev,
                      gs_report* report, double* grad_dev, gs_stats* stats);
bool context_is_multi(const gs_ctx* c);
cudaStream_t context_stream(const gs_ctx* c);
void host_box(const double* q, int64_t n, double* box);

}  // namespace gsb
