// capi.cu -- the C ABI (include/geoshoot_b200.h): contexts, device-resident
// flows, and the reference-facing entry points (kernel_exact / octree /
// bh_kernel / shooting). Host code only orchestrates: every arithmetic step
// of the hot path runs in the sm_100a kernels of allpairs.cu, epilogue.cu,
// tree.cu and bh.cu. There is no CPU fallback -- without a B200 the context
// cannot be created.
#include <chrono>
#include <cstring>
#include <memory>
#include <mutex>
#include <unordered_set>
#include <vector>

#include "bh.h"
#include "engine.h"

namespace gsb {

thread_local std::string g_err;
thread_local KTimer* g_ktimer = nullptr;
thread_local int g_nonfinite = 0;
thread_local uint32_t g_violations = 0;

void set_error(const std::string& msg) { g_err = msg; }

int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  std::snprintf(buf, sizeof buf, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
                cudaGetErrorString(e), what, file, line);
  g_err = buf;
  return GS_CUDA_ERROR;
}

std::atomic<unsigned long long> g_dbuf_epoch{0};

int DBuf::ensure(size_t need) {
  if (need <= bytes && ptr) return GS_OK;
  release();
  ++g_dbuf_epoch;
  need = std::max<size_t>(need, 256);
  GS_CUDA_OK(cudaMalloc(&ptr, need));
  bytes = need;
  return GS_OK;
}

void DBuf::release() {
  if (ptr) {
    cudaFree(ptr);
    ++g_dbuf_epoch;
  }
  ptr = nullptr;
  bytes = 0;
}

}  // namespace gsb

using namespace gsb;

#define GS_TRY(expr)                 \
  do {                               \
    const int s__ = (expr);          \
    if (s__ != GS_OK) return (gs_status)s__; \
  } while (0)

// ----------------------------------------------------------------------------
// context
// ----------------------------------------------------------------------------
struct gs_ctx {
  Device dev;
  cudaStream_t stream = nullptr;
  int lmd = 0;  // gs_set_literal_mean_dot (tree-level Barnes-Hut calls)
  // host-array staging (double [n][3]) and small scalars
  DBuf stage_a, stage_b, stage_c, stage_d, scal;
  DBuf rec_a, rec_b, part, epart;
  gs_flow* scratch = nullptr;
  // caller-owned flows and trees made on this context: gs_destroy detaches
  // them (their ctx becomes null) so that destroying them afterwards only
  // frees their device memory instead of touching a dead context
  std::unordered_set<gs_flow*> flows;
  std::unordered_set<gs_tree*> trees;
  // multi-device context (gs_create_multi): one sub-context (device, stream,
  // workspaces) per target shard; shooting calls shard across them
  std::vector<gs_ctx*> subs;
  bool peer_stores = true;  // epilogues store into peers' buffers (else peer copies)
  std::vector<cudaEvent_t> ev;  // per-shard stage-completion events
  KTimer* timer = nullptr;      // gs_profile: event timing inside shooting calls
};

struct gs_flow {
  gs_ctx* ctx = nullptr;
  gs_config cfg{};
  int prec = kF64;
  int64_t n = 0, shard_begin = 0, shard_count = 0;
  KernelConsts kc{};
  DBuf rec, rec_next, y, ks, part, dhdp0, epart, flags, scal;
  DBuf boxes;  // exact underflow cutoff: target-block and source-tile boxes
  // Barnes-Hut shards: records are put in Morton order once (set_shard) so a
  // shard's index range is a compact region; order[t] = original index of t
  DBuf order;
  bool permuted = false;
  int steps_done = 0;
  int64_t launches = 0;
  bool want_energy = false;
  bool have_energy_part = false;
  int energy_blocks = 0;
  BhWork bh;
  gs_stats stats{};
  KTimer* timer = nullptr;  // gs_flow_profile
  // multi-device flow: one sub-flow per shard (on the sub-contexts); the
  // records ping-pong between rec and rec_next, each stage epilogue storing
  // its shard into every sub-flow's rec_next (PeerOut)
  std::vector<gs_flow*> subs;
  PeerOut peers;     // set by the multi-device driver for the next stage
  int plan_tgt = -1; // exact RHS planned for this many targets (bitwise shards)
  // multi-GPU symmetric exact stages (gs_flow_set_pair_rows): this rank's
  // tile-pair rows, and its per-target fold of them (n x 2 float4)
  int pair_rank = -1, pair_world = 0;
  DBuf pair_out, pair_in;  // (pair_in: a multi-device shard's gathered partials)
  // CUDA graph of one integrator step (all stages + the step-counter bump),
  // captured after the first eager step and replayed for the following ones
  DBuf stepctr;
  cudaGraphExec_t gexec = nullptr;
  KernelConsts gkc{};
  gs_config gcfg{};
  int64_t gn = -1, glaunches = 0;
  unsigned long long gepoch = 0;  // g_dbuf_epoch at capture
  uint64_t gsig = 0;              // the flow's buffer pointers at capture
  void drop_graph() {
    if (gexec) cudaGraphExecDestroy(gexec);
    gexec = nullptr;
  }
  ~gs_flow();
};

gs_flow::~gs_flow() {
  drop_graph();
  delete timer;
  for (gs_flow* s : subs) {
    if (s->ctx) cudaSetDevice(s->ctx->dev.id);
    delete s;
  }
}

static void detach_trees(gs_ctx* c);  // after struct gs_tree

extern "C" {

gs_status gs_set_bh_walk(int32_t kernel, int32_t windows) {
  if (!(kernel == -1 || kernel == 0 || kernel == 1 || kernel == 3 || kernel == 4) || windows < -1 ||
      windows > 64)
    return GS_INVALID_ARGUMENT;
  set_bh_walk(kernel, windows);
  return GS_OK;
}

gs_status gs_set_exact_pairs(int32_t mode) {
  if (mode < -1 || mode > 2) return GS_INVALID_ARGUMENT;
  set_exact_pairs(mode);
  return GS_OK;
}

gs_status gs_set_literal_mean_dot(gs_ctx* c, int32_t enable) {
  if (!c) return GS_INVALID_ARGUMENT;
  c->lmd = enable ? 1 : 0;
  return GS_OK;
}

gs_config gs_default_config(void) {
  gs_config c;
  c.sigma = 2.0;
  c.lambda = 1.0;
  c.timesteps = 40;
  c.backend = GS_EXACT;
  c.threshold_multiplier = 3.0;
  c.integrator = GS_EULER;
  c.precision = GS_F64;
  c.literal_mean_dot = 0;
  c.flags = 0;
  return c;
}

int gs_abi_version(void) { return GS_ABI_VERSION; }

gs_ctx* gs_create(int device, gs_status* status) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0 || device < 0 || device >= count) {
    g_err = std::string("no CUDA device available: ") +
            (e != cudaSuccess ? cudaGetErrorString(e) : "device index out of range");
    if (status) *status = GS_NO_DEVICE;
    return nullptr;
  }
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  if (prop.major < 10) {
    g_err = "geoshoot_b200 needs an sm_100a (Blackwell) device";
    if (status) *status = GS_NO_DEVICE;
    return nullptr;
  }
  cudaSetDevice(device);
  gs_ctx* c = new gs_ctx;
  c->dev.id = device;
  c->dev.sms = prop.multiProcessorCount;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    g_err = "cudaStreamCreate failed";
    delete c;
    if (status) *status = GS_CUDA_ERROR;
    return nullptr;
  }
  if (status) *status = GS_OK;
  return c;
}

void gs_destroy(gs_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->dev.id);
  cudaStreamSynchronize(ctx->stream);
  for (gs_flow* f : ctx->flows) f->ctx = nullptr;
  detach_trees(ctx);
  if (ctx->scratch) gs_flow_destroy(ctx->scratch);
  for (gs_ctx* s : ctx->subs) {  // multi-device: the shards' contexts
    cudaSetDevice(s->dev.id);
    cudaStreamSynchronize(s->stream);
  }
  for (cudaEvent_t e : ctx->ev) cudaEventDestroy(e);
  for (gs_ctx* s : ctx->subs) gs_destroy(s);
  cudaSetDevice(ctx->dev.id);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamDestroy(ctx->stream);
  delete ctx->timer;
  delete ctx;
}

const char* gs_last_error(const gs_ctx*) { return g_err.c_str(); }
int gs_last_nonfinite_step(const gs_ctx*) { return g_nonfinite; }
uint32_t gs_last_config_violations(const gs_ctx*) { return g_violations; }

gs_status gs_validate_config(const gs_config* cfg, uint32_t* mask) {
  uint32_t m = 0;
  if (!(cfg->sigma > 0.0)) m |= GS_VIOLATION_NON_POSITIVE_SIGMA;
  if (!(cfg->lambda > 0.0)) m |= GS_VIOLATION_NON_POSITIVE_LAMBDA;
  if (cfg->timesteps < 1) m |= GS_VIOLATION_ZERO_TIMESTEPS;
  if (!(cfg->threshold_multiplier > 0.0)) m |= GS_VIOLATION_NON_POSITIVE_THRESHOLD;
  if (mask) *mask = m;
  g_violations = m;
  if (m) {
    g_err = "invalid shooting config";
    return GS_CONFIG_ERROR;
  }
  return GS_OK;
}

}  // extern "C"

// ----------------------------------------------------------------------------
// helpers
// ----------------------------------------------------------------------------
namespace {

gs_status bad_arg(const char* msg) {
  g_err = msg;
  return GS_INVALID_ARGUMENT;
}

// host [n][3] doubles -> device staging buffer
int h2d(gs_ctx* c, DBuf& dst, const double* src, int64_t n) {
  GS_TRY(dst.ensure(sizeof(double) * 3 * std::max<int64_t>(n, 1)));
  if (n > 0)
    GS_CUDA_OK(cudaMemcpyAsync(dst.ptr, src, sizeof(double) * 3 * n, cudaMemcpyHostToDevice,
                               c->stream));
  return GS_OK;
}

int d2h(gs_ctx* c, double* dst, const void* src, int64_t count) {
  if (dst && count > 0)
    GS_CUDA_OK(cudaMemcpyAsync(dst, src, sizeof(double) * count, cudaMemcpyDeviceToHost,
                               c->stream));
  return GS_OK;
}

int sync(gs_ctx* c) {
  GS_CUDA_OK(cudaStreamSynchronize(c->stream));
  return GS_OK;
}

// FP32 centring: midpoint of the host bounding box (cheap, keeps |x'| small).
void bbox_center(const double* q, int64_t n, double* c0, double* ext = nullptr) {
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) lo[a] = hi[a] = q[a];
  for (int64_t i = 1; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      const double v = q[3 * i + a];
      lo[a] = v < lo[a] ? v : lo[a];
      hi[a] = v > hi[a] ? v : hi[a];
    }
  for (int a = 0; a < 3; ++a) c0[a] = 0.5 * (lo[a] + hi[a]);
  if (ext)
    for (int a = 0; a < 3; ++a) ext[a] = hi[a] - lo[a];
}

KernelConsts with_ext(KernelConsts k, const double* ext) {
  for (int a = 0; a < 3; ++a) k.ext[a] = ext[a];
  return k;
}

// upload + pack; flags non-finite input (PointSet/MomentumSet ctor, core.hpp:124-170)
int upload_records(gs_ctx* c, int prec, const double* q, const double* p, int64_t n, DBuf& rec) {
  GS_TRY(h2d(c, c->stage_a, q, n));
  if (p) GS_TRY(h2d(c, c->stage_b, p, n));
  GS_TRY(rec.ensure(2 * vec_bytes(prec) * n));
  GS_TRY(c->scal.ensure(64));
  int* bad = c->scal.as<int>();
  GS_CUDA_OK(cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
  GS_TRY(pack_records(prec, c->stage_a.as<double>(), p ? c->stage_b.as<double>() : nullptr, n,
                      rec.ptr, bad, c->stream));
  int hbad = 0;
  GS_CUDA_OK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  GS_TRY(sync(c));
  if (hbad) return bad_arg("non-finite coordinate in input");
  return GS_OK;
}

double fwd_cq(int prec, const KernelConsts& kc) {
  // dH/dq = -(2/s) sum c d ; FP32 partials hold d' = kappa d
  return prec == kF32 ? -kc.two_over_s / kc.kappa : -kc.two_over_s;
}

// FP32 underflow radius of the scaled Gaussian 2^(-r'^2): beyond r'^2 = 150
// every weight is exactly 0; 160 leaves margin for the FP32 box arithmetic.
constexpr float kExactCut2 = 160.0f;

// one exact FP32 RHS over Morton-ordered points (GS_FLAG_EXACT_CUTOFF /
// GS_FLAG_EXACT_MORTON) for all n targets + its epilogue
int exact_sorted_stage(const Device& dev, const KernelConsts& kc, const void* rec, int64_t n,
                       DevTree& t, DBuf& part, DBuf& boxes, bool skip, FwdEpi e,
                       cudaStream_t st, int64_t* launches, int* energy_blocks) {
  GS_TRY(part.ensure((size_t)kMaxChunks * 2 * sizeof(float4) * std::max<int64_t>(n, 1)));
  GS_TRY(morton_order(dev, kF32, kc, rec, n, t, st));
  kt_mark(0, st);
  const int S = rhs_sorted_partials(dev, t.srec.ptr, t.perm.as<int>(), (int)n, part.ptr,
                                    kMaxChunks, boxes, skip ? kExactCut2 : INFINITY, st);
  kt_mark(0, st);
  if (S < 0) { set_error("chunk plan overflow"); return GS_INTERNAL; }
  GS_CUDA_OK(cudaGetLastError());
  e.S = S;
  e.part = part.ptr;
  e.n_tgt = (int)n;
  e.tgt_begin = 0;
  e.cp = 2.0;
  e.cq = fwd_cq(kF32, kc);
  GS_TRY(fwd_epilogue(kF32, e, st, energy_blocks));
  if (launches) *launches += 33;  // Morton order (~28) + boxes (2) + RHS + epilogue
  return GS_OK;
}

// one exact RHS over all n sources for targets [tb, tb + nt) + its epilogue
int exact_stage(const Device& dev, int prec, const KernelConsts& kc, const void* rec, int64_t n,
                int64_t tb, int64_t nt, DBuf& part, FwdEpi e, cudaStream_t st, int64_t* launches,
                int* energy_blocks, int plan_tgt = -1) {
  const bool sym = use_sym(prec, (int)n, (int)tb, (int)nt, plan_tgt);
  const bool sym64 = prec == kF64 && use_sym_f64((int)n, (int)tb, (int)nt, plan_tgt);
  if (sym)
    GS_TRY(part.ensure(sym_part_bytes((int)n)));
  else if (sym64)
    GS_TRY(part.ensure(sym_f64_part_bytes((int)n)));
  else
    GS_TRY(part.ensure((size_t)kMaxChunks * 2 * vec_bytes(prec) * std::max<int64_t>(nt, 1)));
  kt_mark(0, st);
  const int S = sym     ? rhs_sym_partials(rec, (int)n, kc, part.ptr, st)
                : sym64 ? rhs_sym_f64_partials(rec, (int)n, kc, part.ptr, st)
                        : rhs_partials(dev, prec, rec, (int)n, (int)tb, (int)nt, kc, part.ptr,
                                       kMaxChunks, st, plan_tgt);
  kt_mark(0, st);
  if (S < 0) { set_error("chunk plan overflow"); return GS_INTERNAL; }
  GS_CUDA_OK(cudaGetLastError());
  e.S = S;
  e.part = part.ptr;
  e.n_tgt = (int)nt;
  e.tgt_begin = (int)tb;
  e.cp = 2.0;
  e.cq = fwd_cq(prec, kc);
  GS_TRY(fwd_epilogue(prec, e, st, energy_blocks));
  if (launches) *launches += sym64 ? 1 + sym_f64_launches((int)n) : sym ? 1 + sym_launches((int)n) : 2;
  return GS_OK;
}

int check_n(int64_t n) {
  if (n < 1) return bad_arg("point set must contain at least one point");
  if (n > (int64_t)INT32_MAX / 4) return bad_arg("point count exceeds the 2^29 limit");
  return GS_OK;
}

}  // namespace

// ----------------------------------------------------------------------------
// flows
// ----------------------------------------------------------------------------
namespace {

int flow_stages(const gs_flow* f) { return f->cfg.integrator == GS_RK4 ? 4 : 1; }

// Makes t (if any) the thread's kernel timer for a scope (gs_flow_profile,
// gs_profile); a null t keeps the enclosing one.
struct TimerInstall {
  KTimer* prev;
  explicit TimerInstall(KTimer* t) : prev(g_ktimer) {
    if (t) g_ktimer = t;
  }
  ~TimerInstall() { g_ktimer = prev; }
};

// One integrator stage for the shard: RHS (exact or Barnes-Hut) + epilogue.
// rec_in (default: the flow's records) holds all n source records; the
// shard's updated records go to rec_out (default: in place).
// The stage epilogue's parameters for the flow's shard (flow_stage and the
// multi-GPU symmetric stage, gs_flow_stage_apply); *first: this stage also
// forms the energy term (step 0, stage 0).
int flow_epi(gs_flow* f, int stage, void* rec_in, void* rec_out, FwdEpi& e, bool& first) {
  GS_TRY(f->flags.ensure(64));
  e.rec = rec_in;
  e.rec_out = rec_out;
  e.y = f->y.ptr;
  e.ks = f->ks.ptr;
  e.integrator = f->cfg.integrator;
  e.stage = stage;
  e.update = 1;
  e.dt = 1.0 / f->cfg.timesteps;
  e.bad_step = f->flags.as<int>();
  e.step = f->steps_done + 1;
  e.step_dev = f->stepctr.as<int>();
  if (stage == flow_stages(f) - 1) e.step_inc = f->stepctr.as<int>();
  e.peers = f->peers;
  first = f->want_energy && f->steps_done == 0 && stage == 0;
  if (first) {
    GS_TRY(f->epart.ensure(sizeof(double) * (f->shard_count / 128 + 8)));
    GS_TRY(f->dhdp0.ensure(sizeof(double) * 3 * f->shard_count));
    e.energy_part = f->epart.as<double>();
    e.dhdp_out = f->dhdp0.as<double>();
  }
  return GS_OK;
}

int flow_stage(gs_flow* f, int stage, void* rec_in, void* rec_out) {
  gs_ctx* c = f->ctx;
  cudaStream_t st = c->stream;
  if (!rec_in) rec_in = f->rec.ptr;
  FwdEpi e;
  bool first = false;
  GS_TRY(flow_epi(f, stage, rec_in, rec_out, e, first));
  int blocks = 0;
  TimerInstall install(f->timer);
  const bool sorted = f->cfg.backend == GS_EXACT && f->prec == kF32 &&
                      (f->cfg.flags & (GS_FLAG_EXACT_CUTOFF | GS_FLAG_EXACT_MORTON)) &&
                      f->shard_begin == 0 && f->shard_count == f->n;
  if (sorted) {
    GS_TRY(exact_sorted_stage(c->dev, f->kc, rec_in, f->n, f->bh.cur, f->part, f->boxes,
                              (f->cfg.flags & GS_FLAG_EXACT_CUTOFF) != 0, e, st, &f->launches,
                              &blocks));
    f->stats.direct_interactions += (uint64_t)f->n * (uint64_t)f->shard_count;
    f->stats.traversal_queries += (uint64_t)f->shard_count;
  } else if (f->cfg.backend == GS_EXACT) {
    GS_TRY(exact_stage(c->dev, f->prec, f->kc, rec_in, f->n, f->shard_begin, f->shard_count,
                       f->part, e, st, &f->launches, &blocks, f->plan_tgt));
    f->stats.direct_interactions += (uint64_t)f->n * (uint64_t)f->shard_count;
    f->stats.traversal_queries += (uint64_t)f->shard_count;
  } else {
    GS_TRY(bh_forward_stage(c->dev, f->prec, f->kc, f->cfg, rec_in, f->n, f->shard_begin,
                            f->shard_count, f->bh, e, st, &f->launches, &blocks, &f->stats));
  }
  if (first) {
    f->have_energy_part = true;
    f->energy_blocks = blocks;
  }
  return GS_OK;
}

int flow_init(gs_flow* f, gs_ctx* c, const gs_config* cfg, int64_t n) {
  f->ctx = c;
  f->cfg = *cfg;
  f->prec = cfg->precision == GS_F32 ? kF32 : kF64;
  f->n = n;
  f->shard_begin = 0;
  f->shard_count = n;
  f->plan_tgt = -1;
  f->steps_done = 0;
  f->launches = 0;
  f->want_energy = false;
  f->have_energy_part = false;
  f->stats = gs_stats{};
  const size_t rb = 2 * vec_bytes(f->prec) * n;
  GS_TRY(f->rec.ensure(rb));
  if (cfg->integrator == GS_RK4) {
    GS_TRY(f->y.ensure(rb));
    GS_TRY(f->ks.ensure(rb));
  }
  GS_TRY(f->flags.ensure(64));
  GS_CUDA_OK(cudaMemsetAsync(f->flags.ptr, 0x7f, 2 * sizeof(int), c->stream));  // bad_step = +big, no overflow
  GS_TRY(f->bh.stats.ensure(64));
  GS_CUDA_OK(cudaMemsetAsync(f->bh.stats.ptr, 0, 64, c->stream));
  GS_TRY(f->stepctr.ensure(64));
  GS_CUDA_OK(cudaMemsetAsync(f->stepctr.ptr, 0, 2 * sizeof(int), c->stream));
  return GS_OK;
}

// fold the device-side Barnes-Hut counters into the host stats
int flow_bh_stats(gs_flow* f, gs_stats* out) {
  if (f->cfg.backend != GS_BARNES_HUT || !out) return GS_OK;
  unsigned long long v[3] = {0, 0, 0};
  GS_CUDA_OK(cudaMemcpyAsync(v, f->bh.stats.ptr, sizeof v, cudaMemcpyDeviceToHost, f->ctx->stream));
  GS_TRY(sync(f->ctx));
  out->direct_interactions += v[0];
  out->approximated_interactions += v[1];
  out->nodes_visited += v[2];
  return GS_OK;
}

int flow_upload(gs_flow* f, const double* q0, const double* p0) {
  double c0[3], ext[3];
  bbox_center(q0, f->n, c0, ext);
  f->kc = with_ext(make_consts(f->cfg.sigma, f->prec == kF32 ? c0 : nullptr), ext);
  GS_TRY(upload_records(f->ctx, f->prec, q0, p0, f->n, f->rec));
  f->permuted = false;
  f->steps_done = 0;
  f->have_energy_part = false;
  GS_CUDA_OK(cudaMemsetAsync(f->flags.ptr, 0x7f, 2 * sizeof(int), f->ctx->stream));
  GS_CUDA_OK(cudaMemsetAsync(f->stepctr.ptr, 0, 2 * sizeof(int), f->ctx->stream));
  return GS_OK;
}

int flow_step_eager(gs_flow* f) {
  for (int s = 0; s < flow_stages(f); ++s) GS_TRY(flow_stage(f, s, nullptr, nullptr));
  ++f->steps_done;
  return GS_OK;
}

bool graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GS_GRAPHS");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

// Capture one step (the kernel parameters -- buffers, constants -- are fixed
// for a given flow configuration and input scaling), instantiate, keep.
// Every device buffer a captured step can touch: a graph replays raw pointers.
uint64_t flow_sig(const gs_flow* f) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const DBuf& b) {
    h = (h ^ (uint64_t)(uintptr_t)b.ptr) * 1099511628211ull;
    h = (h ^ (uint64_t)b.bytes) * 1099511628211ull;
  };
  for (const DBuf* b : {&f->rec, &f->rec_next, &f->y, &f->ks, &f->part, &f->flags, &f->stepctr,
                        &f->boxes, &f->bh.part, &f->bh.stats})
    mix(*b);
  const DevTree& t = f->bh.cur;
  for (const DBuf* b : {&t.key_hi, &t.key_lo, &t.perm, &t.skey_hi, &t.skey_lo, &t.lcp, &t.first,
                        &t.srec, &t.squ, &t.sadj, &t.meta, &t.parent, &t.nchild, &t.lo,
                        &t.hi, &t.cen, &t.mom, &t.nrec, &t.nadj, &t.psum, &t.msum,
                        &t.asum, &t.bsum, &t.root, &t.tmp_k, &t.tmp_v, &t.tmp_v2, &t.hist, &t.tie_scr, &t.tie_buf, &t.klo_flag, &t.bbox_ctr,
                        &t.scan_tmp, &t.scal, &t.outer, &t.parts, &t.start, &t.sm_ctr})
    mix(*b);
  return h;
}

int flow_capture_step(gs_flow* f) {
  f->drop_graph();
  cudaStream_t st = f->ctx->stream;
  const gs_stats saved = f->stats;
  const int64_t l0 = f->launches;
  const int steps_saved = f->steps_done;
  cudaGraph_t g = nullptr;
  GS_CUDA_OK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  int s = GS_OK;
  for (int k = 0; k < flow_stages(f) && s == GS_OK; ++k) s = flow_stage(f, k, nullptr, nullptr);
  const cudaError_t ce = cudaStreamEndCapture(st, &g);
  f->stats = saved;  // nothing ran during capture
  f->steps_done = steps_saved;
  GS_TRY(s);
  GS_CUDA_OK(ce);
  const cudaError_t ie = cudaGraphInstantiate(&f->gexec, g, 0);
  cudaGraphDestroy(g);
  GS_CUDA_OK(ie);
  f->glaunches = f->launches - l0 + 1;
  f->launches = l0;
  f->gepoch = g_dbuf_epoch.load();
  f->gsig = flow_sig(f);
  std::memcpy(&f->gkc, &f->kc, sizeof f->kc);  // byte copies: compared with memcmp
  std::memcpy(&f->gcfg, &f->cfg, sizeof f->cfg);
  f->gn = f->n;
  return GS_OK;
}

int flow_advance(gs_flow* f, int steps) {
  f->launches = 0;
  const bool graphs = graphs_enabled() && !f->timer && !g_ktimer && f->shard_begin == 0 && f->shard_count == f->n;
  for (int k = 0; k < steps; ++k) {
    bool stale = true;
    if (graphs) {
      stale = !f->gexec || f->gn != f->n || std::memcmp(&f->gkc, &f->kc, sizeof f->kc) != 0 ||
              std::memcmp(&f->gcfg, &f->cfg, sizeof f->cfg) != 0;
      if (!stale && f->gepoch != g_dbuf_epoch.load()) {  // some buffer somewhere moved: ours?
        stale = flow_sig(f) != f->gsig;
        if (!stale) f->gepoch = g_dbuf_epoch.load();
      }
    }
    // the first step runs eagerly (its energy term, first-use allocations)
    // unless an earlier run of this flow left a valid graph and no energy is wanted
    if (!graphs || (f->steps_done == 0 && (stale || f->want_energy))) {
      GS_TRY(flow_step_eager(f));
      continue;
    }
    if (stale) GS_TRY(flow_capture_step(f));
    GS_CUDA_OK(cudaGraphLaunch(f->gexec, f->ctx->stream));
    f->launches += f->glaunches;
    ++f->steps_done;
    if (f->cfg.backend == GS_EXACT) {  // the host-side counters an eager step keeps
      f->stats.direct_interactions += (uint64_t)flow_stages(f) * f->n * (uint64_t)f->shard_count;
      f->stats.traversal_queries += (uint64_t)flow_stages(f) * f->shard_count;
    }
  }
  return GS_OK;
}

// returns GS_NONFINITE (and records the step) if the device flag was raised
int flow_check(gs_flow* f) {
  int fl[2] = {0, 0};
  GS_CUDA_OK(cudaMemcpyAsync(fl, f->flags.ptr, sizeof fl, cudaMemcpyDeviceToHost,
                             f->ctx->stream));
  GS_TRY(sync(f->ctx));
  const int bad = fl[0];
  if (fl[1] == 1) {
    g_err = "octree node capacity (4n + 64) exceeded: degenerate point clustering";
    return GS_INTERNAL;
  }
  if (bad != 0x7f7f7f7f) {
    g_nonfinite = bad;
    g_err = "non-finite state at timestep " + std::to_string(bad);
    return GS_NONFINITE;
  }
  return GS_OK;
}

int flow_energy(gs_flow* f, double* out) {
  if (!f->have_energy_part) { *out = 0.0; return GS_OK; }
  GS_TRY(f->scal.ensure(64));
  GS_TRY(reduce_sum(f->epart.as<double>(), f->energy_blocks, f->scal.as<double>(), f->ctx->stream));
  double h = 0.0;
  GS_CUDA_OK(cudaMemcpyAsync(&h, f->scal.ptr, sizeof(double), cudaMemcpyDeviceToHost,
                             f->ctx->stream));
  GS_TRY(sync(f->ctx));
  *out = 0.5 * h;  // H = 1/2 <p0, dH/dp>, shooting.cpp:104-108
  return GS_OK;
}

gs_flow* scratch_flow(gs_ctx* c) {
  if (!c->scratch) c->scratch = new gs_flow;
  return c->scratch;
}

// Barnes-Hut walks are only coherent for spatially compact query sets: a
// sharded flow reorders its records by Morton key once (every shard computes
// the same order from the same uploaded records) and remembers the order for
// download.
int flow_morton_permute(gs_flow* f) {
  gs_ctx* c = f->ctx;
  GS_TRY(morton_order(c->dev, f->prec, f->kc, f->rec.ptr, f->n, f->bh.cur, c->stream));
  GS_TRY(f->order.ensure(sizeof(int) * f->n));
  GS_CUDA_OK(cudaMemcpyAsync(f->order.ptr, f->bh.cur.perm.ptr, sizeof(int) * f->n,
                             cudaMemcpyDeviceToDevice, c->stream));
  GS_TRY(f->rec_next.ensure(2 * vec_bytes(f->prec) * f->n));
  GS_TRY(permute_records(f->prec, f->rec.ptr, f->order.as<int>(), f->n, f->rec_next.ptr, c->stream));
  std::swap(f->rec.ptr, f->rec_next.ptr);
  std::swap(f->rec.bytes, f->rec_next.bytes);
  f->permuted = true;
  return GS_OK;
}

// multi-device contexts (definitions at the end of this file)
bool is_multi(const gs_ctx* c) { return c && !c->subs.empty(); }
int multi_flow_init(gs_flow* f, gs_ctx* c, const gs_config* cfg, int64_t n);
int multi_flow_upload(gs_flow* f, const double* q0, const double* p0);
int multi_flow_advance(gs_flow* f, int steps);
int multi_flow_check(gs_flow* f);
int multi_flow_download(gs_flow* f, double* q, double* p);
int multi_flow_stats(gs_flow* f, gs_stats* out);
int multi_flow_energy(gs_flow* f, double* out);
int multi_evaluate(gs_ctx* c, const gs_config* cfg, int64_t n, const double* q0, const double* p0,
                   const double* target, gs_report* report, double* grad_out, gs_stats* stats);

struct Timer {
  cudaEvent_t a{}, b{};
  cudaStream_t s;
  explicit Timer(cudaStream_t st) : s(st) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  double ms() {
    float v = 0.f;
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&v, a, b);
    return v;
  }
  ~Timer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

}  // namespace

extern "C" {

gs_status gs_flow_create(gs_ctx* ctx, const gs_config* cfg, int64_t n, gs_flow** out) {
  if (!ctx || !cfg || !out) return bad_arg("null argument");
  GS_TRY(gs_validate_config(cfg, nullptr));
  GS_TRY(check_n(n));
  auto* f = new gs_flow;
  const int s = is_multi(ctx) ? multi_flow_init(f, ctx, cfg, n) : flow_init(f, ctx, cfg, n);
  if (s != GS_OK) {
    delete f;
    return (gs_status)s;
  }
  ctx->flows.insert(f);
  *out = f;
  return GS_OK;
}

void gs_flow_destroy(gs_flow* flow) {
  if (!flow) return;
  if (flow->ctx) {
    cudaStreamSynchronize(flow->ctx->stream);
    flow->ctx->flows.erase(flow);
  }
  delete flow;
}

gs_status gs_flow_upload(gs_flow* f, const double* q0, const double* p0) {
  if (!f || !q0 || !p0) return bad_arg("null argument");
  if (!f->subs.empty()) return (gs_status)multi_flow_upload(f, q0, p0);
  return (gs_status)flow_upload(f, q0, p0);
}

gs_status gs_flow_advance(gs_flow* f, int32_t steps) {
  if (!f) return bad_arg("null flow");
  if (!f->subs.empty()) return (gs_status)multi_flow_advance(f, steps);
  return (gs_status)flow_advance(f, steps);
}

gs_status gs_flow_sync(gs_flow* f) {
  if (!f) return bad_arg("null flow");
  if (!f->subs.empty()) return (gs_status)multi_flow_check(f);
  return (gs_status)flow_check(f);
}

gs_status gs_flow_download(gs_flow* f, double* q, double* p) {
  if (!f) return bad_arg("null flow");
  if (!f->subs.empty()) return (gs_status)multi_flow_download(f, q, p);
  gs_ctx* c = f->ctx;
  GS_TRY(c->stage_a.ensure(sizeof(double) * 3 * f->n));
  GS_TRY(c->stage_b.ensure(sizeof(double) * 3 * f->n));
  GS_TRY(unpack_records(f->prec, f->rec.ptr, f->n, c->stage_a.as<double>(),
                        c->stage_b.as<double>(), c->stream));
  if (f->permuted) {  // back to the caller's point order
    GS_TRY(c->stage_c.ensure(sizeof(double) * 3 * f->n));
    GS_TRY(c->stage_d.ensure(sizeof(double) * 3 * f->n));
    GS_TRY(scatter_rows3(c->stage_a.as<double>(), f->order.as<int>(), f->n, c->stage_c.as<double>(), c->stream));
    GS_TRY(scatter_rows3(c->stage_b.as<double>(), f->order.as<int>(), f->n, c->stage_d.as<double>(), c->stream));
    GS_TRY(d2h(c, q, c->stage_c.ptr, 3 * f->n));
    GS_TRY(d2h(c, p, c->stage_d.ptr, 3 * f->n));
  } else {
    GS_TRY(d2h(c, q, c->stage_a.ptr, 3 * f->n));
    GS_TRY(d2h(c, p, c->stage_b.ptr, 3 * f->n));
  }
  GS_TRY(sync(c));
  return GS_OK;
}

int64_t gs_flow_last_launches(const gs_flow* f) { return f ? f->launches : 0; }
void* gs_flow_stream(const gs_flow* f) { return f ? (void*)f->ctx->stream : nullptr; }

gs_status gs_flow_profile(gs_flow* f, int32_t enable) {
  if (!f) return bad_arg("null flow");
  if (!f->subs.empty()) return bad_arg("profiling is per device: not on a multi-device flow");
  if (enable && !f->timer) f->timer = new KTimer;
  if (!enable) {
    delete f->timer;
    f->timer = nullptr;
  }
  return GS_OK;
}

gs_status gs_flow_profile_read(gs_flow* f, double* kernel_ms, int64_t* kernel_launches,
                               double* build_ms, int64_t* builds) {
  if (!f || !f->timer) return bad_arg("profiling not enabled");
  GS_CUDA_OK(cudaStreamSynchronize(f->ctx->stream));
  const double k = f->timer->drain(0, kernel_launches);
  const double b = f->timer->drain(1, builds);
  if (kernel_ms) *kernel_ms = k;
  if (build_ms) *build_ms = b;
  return GS_OK;
}

gs_status gs_flow_profile_phases(gs_flow* f, double* ms, int64_t* counts, int32_t channels) {
  if (!f || !f->timer) return bad_arg("profiling not enabled");
  GS_CUDA_OK(cudaStreamSynchronize(f->ctx->stream));
  for (int c = 0; c < channels && c < KTimer::kChannels; ++c) ms[c] = f->timer->drain(c, counts + c);
  return GS_OK;
}

gs_status gs_profile(gs_ctx* c, int32_t enable) {
  if (!c) return bad_arg("null context");
  if (enable && !c->timer) c->timer = new KTimer;
  if (!enable) {
    delete c->timer;
    c->timer = nullptr;
  }
  return GS_OK;
}

gs_status gs_profile_phases(gs_ctx* c, double* ms, int64_t* counts, int32_t channels) {
  if (!c || !c->timer) return bad_arg("profiling not enabled");
  GS_CUDA_OK(cudaStreamSynchronize(c->stream));
  for (int k = 0; k < channels && k < KTimer::kChannels; ++k) ms[k] = c->timer->drain(k, counts + k);
  return GS_OK;
}

namespace {
unsigned long long* g_trace_buf = nullptr;  // device: [0] count, then {tag, t} pairs (trace.cuh)
constexpr int64_t kTraceCap = 16384;
}  // namespace

gs_status gs_trace(gs_ctx* c, int32_t enable) {
  if (!c) return bad_arg("null context");
  GS_CUDA_OK(cudaSetDevice(c->dev.id));
  GS_CUDA_OK(cudaStreamSynchronize(c->stream));
  if (enable && !g_trace_buf) {
    GS_CUDA_OK(cudaMalloc(&g_trace_buf, sizeof(unsigned long long) * (1 + 2 * kTraceCap)));
    GS_CUDA_OK(cudaMemset(g_trace_buf, 0, sizeof(unsigned long long)));
  }
  unsigned long long* b = enable ? g_trace_buf : nullptr;
  GS_TRY(trace_install_tree(b));
  GS_TRY(trace_install_bh(b));
  GS_TRY(trace_install_epi(b));
  if (!enable && g_trace_buf) {
    GS_CUDA_OK(cudaFree(g_trace_buf));
    g_trace_buf = nullptr;
  }
  return GS_OK;
}

gs_status gs_trace_read(gs_ctx* c, uint64_t* tags, uint64_t* times_ns, int64_t max, int64_t* count) {
  if (!c || !count || (max > 0 && (!tags || !times_ns))) return bad_arg("null argument");
  if (!g_trace_buf) return bad_arg("tracing not enabled");
  GS_CUDA_OK(cudaStreamSynchronize(c->stream));
  unsigned long long k = 0;
  GS_CUDA_OK(cudaMemcpy(&k, g_trace_buf, sizeof k, cudaMemcpyDeviceToHost));
  const int64_t got = std::min<int64_t>({(int64_t)k, kTraceCap, max});
  std::vector<unsigned long long> h(2 * std::max<int64_t>(got, 1));
  if (got > 0)
    GS_CUDA_OK(cudaMemcpy(h.data(), g_trace_buf + 1, sizeof(unsigned long long) * 2 * got,
                          cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < got; ++i) {
    tags[i] = h[2 * i];
    times_ns[i] = h[2 * i + 1];
  }
  *count = got;
  GS_CUDA_OK(cudaMemset(g_trace_buf, 0, sizeof(unsigned long long)));
  return GS_OK;
}

gs_status gs_flow_stats(gs_flow* f, gs_stats* out) {
  if (!f || !out) return bad_arg("null argument");
  if (!f->subs.empty()) return (gs_status)multi_flow_stats(f, out);
  *out = f->stats;
  GS_TRY(flow_bh_stats(f, out));
  return GS_OK;
}

gs_status gs_flow_set_shard(gs_flow* f, int64_t begin, int64_t count) {
  if (!f || begin < 0 || count < 0 || begin + count > f->n) return bad_arg("bad shard range");
  if (!f->subs.empty()) return bad_arg("a multi-device flow shards itself");
  f->shard_begin = begin;
  f->shard_count = count;
  f->plan_tgt = (int)f->n;  // shards run the full problem's plan: bit-identical sums
  if (f->cfg.backend == GS_BARNES_HUT && count < f->n && !f->permuted && f->steps_done == 0)
    GS_TRY(flow_morton_permute(f));
  return GS_OK;
}

void* gs_flow_source_buffer(gs_flow* f) { return f ? f->rec.ptr : nullptr; }
int64_t gs_flow_record_bytes(const gs_flow* f) { return f ? 2 * (int64_t)vec_bytes(f->prec) : 0; }

gs_status gs_flow_set_pair_rows(gs_flow* f, int32_t rank, int32_t world, int32_t* enabled) {
  if (!f || !enabled || world < 1 || rank < 0 || rank >= world) return bad_arg("bad rank / world");
  if (!f->subs.empty()) return bad_arg("a multi-device flow shards itself");
  const bool ok = f->cfg.backend == GS_EXACT && f->prec == kF32 &&
                  !(f->cfg.flags & (GS_FLAG_EXACT_CUTOFF | GS_FLAG_EXACT_MORTON)) &&
                  use_sym(kF32, (int)f->n, 0, (int)f->n, -1) && !sym_grouped((int)f->n);
  f->pair_rank = ok ? rank : -1;
  f->pair_world = ok ? world : 0;
  *enabled = ok ? 1 : 0;
  return GS_OK;
}

gs_status gs_flow_stage_pairs(gs_flow* f, int32_t stage, void** partials) {
  if (!f || !partials || stage < 0 || stage >= flow_stages(f)) return bad_arg("bad stage");
  if (f->pair_rank < 0) return bad_arg("gs_flow_set_pair_rows has not enabled pair rows");
  gs_ctx* c = f->ctx;
  GS_TRY(f->part.ensure(sym_part_bytes((int)f->n)));
  GS_TRY(f->pair_out.ensure(2 * sizeof(float4) * (size_t)f->n));
  f->launches = 0;
  TimerInstall install(f->timer);
  kt_mark(0, c->stream);
  rhs_sym_rows(f->rec.ptr, (int)f->n, f->kc, f->part.ptr, f->pair_out.ptr, f->pair_rank,
               f->pair_world, c->stream);
  kt_mark(0, c->stream);
  GS_CUDA_OK(cudaGetLastError());
  f->launches += 2;
  *partials = f->pair_out.ptr;
  return GS_OK;
}

gs_status gs_flow_stage_apply(gs_flow* f, int32_t stage, const void* parts, int32_t nparts) {
  if (!f || !parts || nparts < 1 || stage < 0 || stage >= flow_stages(f)) return bad_arg("bad stage");
  if (f->pair_rank < 0) return bad_arg("gs_flow_set_pair_rows has not enabled pair rows");
  gs_ctx* c = f->ctx;
  FwdEpi e;
  bool first = false;
  GS_TRY(flow_epi(f, stage, f->rec.ptr, nullptr, e, first));
  e.S = nparts;
  e.part = parts;
  e.n_tgt = (int)f->shard_count;
  e.tgt_begin = (int)f->shard_begin;
  e.cp = 2.0;
  e.cq = fwd_cq(kF32, f->kc);
  int blocks = 0;
  GS_TRY(fwd_epilogue(kF32, e, c->stream, &blocks));
  f->launches = 1;
  f->stats.direct_interactions += (uint64_t)f->n * (uint64_t)f->shard_count;
  f->stats.traversal_queries += (uint64_t)f->shard_count;
  if (first) {
    f->have_energy_part = true;
    f->energy_blocks = blocks;
  }
  if (stage == flow_stages(f) - 1) ++f->steps_done;
  return GS_OK;
}

gs_status gs_flow_stage(gs_flow* f, int32_t stage) {
  if (!f || stage < 0 || stage >= flow_stages(f)) return bad_arg("bad stage");
  if (!f->subs.empty()) return bad_arg("a multi-device flow advances with gs_flow_advance");
  f->launches = 0;
  GS_TRY(flow_stage(f, stage, nullptr, nullptr));
  if (stage == flow_stages(f) - 1) ++f->steps_done;  // (the epilogue advanced the step counter)
  return GS_OK;
}

// ----------------------------------------------------------------------------
// kernel_exact
// ----------------------------------------------------------------------------
gs_status gs_exact_pairs_plan(int32_t precision, int64_t n, int32_t* tiles) {
  if (!tiles) return bad_arg("null argument");
  GS_TRY(check_n(n));
  const int prec = precision == GS_F32 ? kF32 : kF64;
  if (prec == kF32)
    *tiles = use_sym(prec, (int)n, 0, (int)n, -1) ? sym_tiles((int)n) : 0;
  else
    *tiles = use_sym_f64((int)n, 0, (int)n, -1) ? sym_f64_tiles((int)n) : 0;
  return GS_OK;
}

gs_status gs_exact_rhs(gs_ctx* c, int32_t precision, int64_t n, const double* q, const double* p,
                       double sigma, double* dHdp, double* dHdq, double* h_out) {
  if (!c || !q || !p) return bad_arg("null argument");
  GS_TRY(check_n(n));
  const int prec = precision == GS_F32 ? kF32 : kF64;
  double c0[3], ext[3];
  bbox_center(q, n, c0, ext);
  const KernelConsts kc = with_ext(make_consts(sigma, prec == kF32 ? c0 : nullptr), ext);
  GS_TRY(upload_records(c, prec, q, p, n, c->rec_a));
  GS_TRY(c->stage_c.ensure(sizeof(double) * 3 * n));
  GS_TRY(c->stage_d.ensure(sizeof(double) * 3 * n));
  GS_TRY(c->epart.ensure(sizeof(double) * (n / 128 + 8)));
  GS_TRY(c->scal.ensure(64));
  FwdEpi e;
  e.rec = c->rec_a.ptr;
  e.update = 0;
  e.dhdp_out = c->stage_c.as<double>();
  e.dhdq_out = c->stage_d.as<double>();
  e.energy_part = h_out ? c->epart.as<double>() : nullptr;
  int blocks = 0;
  GS_TRY(exact_stage(c->dev, prec, kc, c->rec_a.ptr, n, 0, n, c->part, e, c->stream, nullptr,
                     &blocks));
  double h = 0.0;
  if (h_out) {
    GS_TRY(reduce_sum(c->epart.as<double>(), blocks, c->scal.as<double>(), c->stream));
    GS_CUDA_OK(cudaMemcpyAsync(&h, c->scal.ptr, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  }
  GS_TRY(d2h(c, dHdp, c->stage_c.ptr, 3 * n));
  GS_TRY(d2h(c, dHdq, c->stage_d.ptr, 3 * n));
  GS_TRY(sync(c));
  if (h_out) *h_out = 0.5 * h;  // H = 1/2 <p, dH/dp> (same double sum, kernel_exact.hpp:22-28)
  return GS_OK;
}

gs_status gs_hamiltonian(gs_ctx* c, int32_t precision, int64_t n, const double* q,
                         const double* p, double sigma, double* h_out) {
  if (!h_out) return bad_arg("null argument");
  return gs_exact_rhs(c, precision, n, q, p, sigma, nullptr, nullptr, h_out);
}

gs_status gs_exact_velocity(gs_ctx* c, int32_t precision, int64_t m, const double* x, int64_t n,
                            const double* q, const double* p, double sigma, double* v_out) {
  if (!c || !x || !q || !p || !v_out) return bad_arg("null argument");
  GS_TRY(check_n(n));
  GS_TRY(check_n(m));
  const int prec = precision == GS_F32 ? kF32 : kF64;
  double c0[3], ext[3];
  bbox_center(q, n, c0, ext);
  const KernelConsts kc = with_ext(make_consts(sigma, prec == kF32 ? c0 : nullptr), ext);
  GS_TRY(upload_records(c, prec, q, p, n, c->rec_a));
  GS_TRY(upload_records(c, prec, x, nullptr, m, c->rec_b));
  GS_TRY(c->part.ensure((size_t)kMaxChunks * vec_bytes(prec) * m));
  GS_TRY(c->stage_c.ensure(sizeof(double) * 3 * m));
  const int S = vel_partials(c->dev, prec, c->rec_a.ptr, (int)n, c->rec_b.ptr, (int)m, kc,
                             c->part.ptr, kMaxChunks, c->stream);
  if (S < 0) return (gs_status)GS_INTERNAL;
  GS_CUDA_OK(cudaGetLastError());
  VelEpi e;
  e.m = (int)m;
  e.S = S;
  e.part = c->part.ptr;
  e.scale = 1.0;
  e.v_out = c->stage_c.as<double>();
  GS_TRY(vel_epilogue(prec, e, c->stream));
  GS_TRY(d2h(c, v_out, c->stage_c.ptr, 3 * m));
  GS_TRY(sync(c));
  return GS_OK;
}

gs_status gs_hessian_products(gs_ctx* c, int32_t precision, int64_t n, const double* q,
                              const double* p, const double* alpha, const double* beta,
                              double sigma, double* pq, double* pp, double* qq, double* qp) {
  if (!c || !q || !p || !alpha || !beta) return bad_arg("null argument");
  GS_TRY(check_n(n));
  const int prec = precision == GS_F32 ? kF32 : kF64;
  double c0[3], ext[3];
  bbox_center(q, n, c0, ext);
  const KernelConsts kc = with_ext(make_consts(sigma, prec == kF32 ? c0 : nullptr), ext);
  GS_TRY(upload_records(c, prec, q, p, n, c->rec_a));
  GS_TRY(upload_records(c, prec, alpha, beta, n, c->rec_b));
  GS_TRY(c->part.ensure(hess_part_bytes(prec, (int)n, 0, (int)n)));
  DBuf* outs[4] = {&c->stage_a, &c->stage_b, &c->stage_c, &c->stage_d};
  for (DBuf* b : outs) GS_TRY(b->ensure(sizeof(double) * 3 * n));
  const int S = hess_partials(c->dev, prec, c->rec_a.ptr, c->rec_b.ptr, (int)n, 0, (int)n, kc,
                              c->part.ptr, kMaxChunks, c->stream);
  if (S < 0) return (gs_status)GS_INTERNAL;
  GS_CUDA_OK(cudaGetLastError());
  BwdEpi e;
  e.n_tgt = (int)n;
  e.S = S;
  e.part = c->part.ptr;
  e.update = 0;
  const double cd = prec == kF32 ? kc.two_over_s / kc.kappa : kc.two_over_s;
  e.cpq = -cd;
  e.cpp = 2.0;
  e.cqq = kc.two_over_s;
  e.cqp = -cd;
  for (int k = 0; k < 4; ++k) e.out[k] = outs[k]->as<double>();
  GS_TRY(bwd_epilogue(prec, e, c->stream));
  double* hs[4] = {pq, pp, qq, qp};
  for (int k = 0; k < 4; ++k) GS_TRY(d2h(c, hs[k], outs[k]->ptr, 3 * n));
  GS_TRY(sync(c));
  return GS_OK;
}

// ----------------------------------------------------------------------------
// shooting
// ----------------------------------------------------------------------------
gs_status gs_shoot_forward(gs_ctx* c, const gs_config* cfg, int64_t n, const double* q0,
                           const double* p0, double* traj_q, double* traj_p, double* final_q,
                           double* final_p, double* energy_out, gs_stats* stats) {
  if (!c || !cfg || !q0 || !p0) return bad_arg("null argument");
  TimerInstall install(c->timer);
  GS_TRY(gs_validate_config(cfg, nullptr));
  GS_TRY(check_n(n));
  gs_flow* f = scratch_flow(c);
  if (is_multi(c)) {  // target shards across the context's devices
    GS_TRY(multi_flow_init(f, c, cfg, n));
    for (gs_flow* s : f->subs) s->want_energy = energy_out != nullptr;
    GS_TRY(multi_flow_upload(f, q0, p0));
    const int T = cfg->timesteps;
    const auto t0 = std::chrono::steady_clock::now();
    for (int k = 0; k <= T; ++k) {
      if (traj_q || traj_p) {
        std::vector<double> tq((size_t)3 * n), tp((size_t)3 * n);
        GS_TRY(multi_flow_download(f, tq.data(), tp.data()));
        if (traj_q) std::memcpy(traj_q + (size_t)3 * n * k, tq.data(), sizeof(double) * 3 * n);
        if (traj_p) std::memcpy(traj_p + (size_t)3 * n * k, tp.data(), sizeof(double) * 3 * n);
        if (k < T) GS_TRY(multi_flow_advance(f, 1));
      } else if (k == 0) {
        GS_TRY(multi_flow_advance(f, T));
      }
    }
    GS_TRY(multi_flow_check(f));
    const double fwd_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (final_q || final_p) {
      std::vector<double> fq((size_t)3 * n), fp((size_t)3 * n);
      GS_TRY(multi_flow_download(f, fq.data(), fp.data()));
      if (final_q) std::memcpy(final_q, fq.data(), sizeof(double) * 3 * n);
      if (final_p) std::memcpy(final_p, fp.data(), sizeof(double) * 3 * n);
    }
    if (energy_out) GS_TRY(multi_flow_energy(f, energy_out));
    if (stats) {
      GS_TRY(multi_flow_stats(f, stats));
      stats->forward_ms = fwd_ms;
    }
    return GS_OK;
  }
  GS_TRY(flow_init(f, c, cfg, n));
  GS_TRY(flow_upload(f, q0, p0));
  f->want_energy = energy_out != nullptr;
  const int T = cfg->timesteps;
  const bool traj = traj_q || traj_p;
  if (traj) {
    GS_TRY(c->stage_c.ensure(sizeof(double) * 3 * n * (T + 1)));
    GS_TRY(c->stage_d.ensure(sizeof(double) * 3 * n * (T + 1)));
  }
  Timer tm(c->stream);
  if (!traj) {
    GS_TRY(flow_advance(f, T));  // graph-replayed after the first step
  } else {
    for (int k = 0; k <= T; ++k) {
      GS_TRY(unpack_records(f->prec, f->rec.ptr, n, c->stage_c.as<double>() + (size_t)3 * n * k,
                            c->stage_d.as<double>() + (size_t)3 * n * k, c->stream));
      if (k < T) GS_TRY(flow_step_eager(f));
    }
  }
  const double fwd_ms = tm.ms();
  GS_TRY(flow_check(f));
  if (traj) {
    GS_TRY(d2h(c, traj_q, c->stage_c.ptr, 3 * n * (T + 1)));
    GS_TRY(d2h(c, traj_p, c->stage_d.ptr, 3 * n * (T + 1)));
  }
  if (final_q || final_p) {
    GS_TRY(c->stage_a.ensure(sizeof(double) * 3 * n));
    GS_TRY(c->stage_b.ensure(sizeof(double) * 3 * n));
    GS_TRY(unpack_records(f->prec, f->rec.ptr, n, c->stage_a.as<double>(), c->stage_b.as<double>(),
                          c->stream));
    GS_TRY(d2h(c, final_q, c->stage_a.ptr, 3 * n));
    GS_TRY(d2h(c, final_p, c->stage_b.ptr, 3 * n));
  }
  GS_TRY(sync(c));
  if (energy_out) GS_TRY(flow_energy(f, energy_out));
  if (stats) {
    *stats = f->stats;
    GS_TRY(flow_bh_stats(f, stats));
    stats->forward_ms = fwd_ms - f->stats.tree_build_ms;
  }
  return GS_OK;
}

}  // extern "C"

namespace {

// One adjoint step k (shooting.cpp:177-214) for targets [tb, tb + nt): the
// Hessian products of state rk against the full adjoints adj_in, then
// alpha += dt (pq - qq), beta += dt (pp - qp) into e.adj_out (in place if
// null; plus e.peers on a multi-device context).
int backward_step(gs_ctx* c, const gs_config* cfg, int prec, const KernelConsts& kc, int64_t n,
                  int64_t tb, int64_t nt, const void* rk, void* adj_in, int k, BhWork* bh,
                  bool trees_cached, DBuf& part, BwdEpi e, gs_stats* stats, int plan_tgt = -1) {
  cudaStream_t st = c->stream;
  e.n_tgt = (int)nt;
  e.tgt_begin = (int)tb;
  e.adj = adj_in;
  if (cfg->backend == GS_EXACT) {
    GS_TRY(part.ensure(hess_part_bytes(prec, (int)n, (int)tb, (int)nt, plan_tgt)));
    kt_mark(6, st);
    const int S = hess_partials(c->dev, prec, rk, adj_in, (int)n, (int)tb, (int)nt, kc, part.ptr,
                                kMaxChunks, st, plan_tgt);
    kt_mark(6, st);
    if (S < 0) return GS_INTERNAL;
    GS_CUDA_OK(cudaGetLastError());
    e.S = S;
    e.part = part.ptr;
    GS_TRY(bwd_epilogue(prec, e, st));
    if (stats) {
      stats->direct_interactions += (uint64_t)n * nt;
      stats->traversal_queries += nt;
    }
    return GS_OK;
  }
  return bh_backward_step(c->dev, prec, kc, *cfg, rk, adj_in, n, tb, nt, k, *bh, trees_cached, e,
                          st, stats);
}

// Adjoint recursion over device-resident trajectory records traj[0..T]
// (run_backward, shooting.cpp:143-240). dhdp0 must hold dH/dp(q0, p0).
int backward_pass(gs_ctx* c, const gs_config* cfg, int prec, const KernelConsts& kc, int64_t n,
                  const char* traj, size_t rec_bytes, const double* target_dev,
                  const double* dhdp0, BhWork* bh, bool trees_cached, DBuf& adj, DBuf& part,
                  double* grad_dev, double* sse_dev, gs_stats* stats) {
  cudaStream_t st = c->stream;
  const int T = cfg->timesteps;
  const double dt = 1.0 / T;
  GS_TRY(adj.ensure(rec_bytes));
  GS_TRY(c->epart.ensure(sizeof(double) * (n / 128 + 8)));
  int blocks = 0;
  GS_TRY(adjoint_init(prec, traj + (size_t)T * rec_bytes, target_dev, cfg->lambda, n, adj.ptr,
                      c->epart.as<double>(), &blocks, st));
  if (sse_dev) GS_TRY(reduce_sum(c->epart.as<double>(), blocks, sse_dev, st));
  const double cd = prec == kF32 ? kc.two_over_s / kc.kappa : kc.two_over_s;
  BwdEpi e;
  e.n_tgt = (int)n;
  e.adj = adj.ptr;
  e.update = 1;
  e.dt = dt;
  e.cpq = -cd;
  e.cpp = 2.0;
  e.cqq = kc.two_over_s;
  e.cqp = -cd;
  for (int k = T - 1; k >= 0; --k)
    GS_TRY(backward_step(c, cfg, prec, kc, n, 0, n, traj + (size_t)k * rec_bytes, adj.ptr, k, bh,
                         trees_cached, part, e, stats));
  GS_TRY(gradient_finalize(prec, adj.ptr, dhdp0, n, grad_dev, st));
  return GS_OK;
}

}  // namespace

extern "C" {

}  // extern "C"

namespace gsb {

// evaluate() (shooting.cpp:302-314) with the inputs either on the host
// (gs_evaluate) or already resident in HBM (the device optimizer:
// evaluate_resident): q0, p0, target double [n][3]; `box` = the host bounding
// box {c0[3], ext[3]} of q0 (its kernel constants). The gradient goes to the
// host (grad_host) or stays in HBM (grad_dev).
static int evaluate_impl(gs_ctx* c, const gs_config* cfg, int64_t n, const double* q0,
                         const double* p0, const double* target, bool resident, const double* box,
                         gs_report* report, double* grad_host, double* grad_dev, gs_stats* stats) {
  const int T = cfg->timesteps;
  gs_flow* f = scratch_flow(c);
  GS_TRY(flow_init(f, c, cfg, n));
  if (resident) {  // records packed straight from the device arrays
    f->kc = with_ext(make_consts(cfg->sigma, f->prec == kF32 ? box : nullptr), box + 3);
    GS_TRY(c->scal.ensure(64));
    int* bad = c->scal.as<int>();
    GS_CUDA_OK(cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
    GS_TRY(pack_records(f->prec, q0, p0, n, f->rec.ptr, bad, c->stream));
    int hbad = 0;
    GS_CUDA_OK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    GS_TRY(sync(c));
    if (hbad) return bad_arg("non-finite coordinate in input");
    f->permuted = false;
    f->steps_done = 0;
    f->have_energy_part = false;
    GS_CUDA_OK(cudaMemsetAsync(f->flags.ptr, 0x7f, 2 * sizeof(int), c->stream));
    GS_CUDA_OK(cudaMemsetAsync(f->stepctr.ptr, 0, 2 * sizeof(int), c->stream));
  } else {
    GS_TRY(flow_upload(f, q0, p0));
    GS_TRY(h2d(c, c->stage_c, target, n));
    target = c->stage_c.as<double>();
  }
  f->want_energy = true;
  const size_t rb = 2 * vec_bytes(f->prec) * n;
  // trajectory records traj[0..T] resident in HBM
  GS_TRY(c->rec_b.ensure(rb * (T + 1)));
  char* traj = c->rec_b.as<char>();
  GS_CUDA_OK(cudaMemcpyAsync(traj, f->rec.ptr, rb, cudaMemcpyDeviceToDevice, c->stream));
  if (cfg->backend == GS_BARNES_HUT) GS_TRY(bh_keep_trees(f->bh, T));
  Timer tf(c->stream);
  for (int k = 0; k < T; ++k) {
    // RHS reads traj[k]; the epilogue writes traj[k+1]
    f->bh.cache_slot = cfg->backend == GS_BARNES_HUT ? k : -1;
    const int s = flow_stage(f, 0, traj + (size_t)k * rb, traj + (size_t)(k + 1) * rb);
    f->bh.cache_slot = -1;
    GS_TRY(s);
    ++f->steps_done;
  }
  const double fwd_ms = tf.ms();
  GS_TRY(flow_check(f));
  double energy = 0.0;
  GS_TRY(flow_energy(f, &energy));
  if (!grad_dev) {
    GS_TRY(c->stage_d.ensure(sizeof(double) * 3 * n));
    grad_dev = c->stage_d.as<double>();
  }
  GS_TRY(c->scal.ensure(64));
  gs_stats bst{};
  Timer tb(c->stream);
  GS_TRY(backward_pass(c, cfg, f->prec, f->kc, n, traj, rb, target, f->dhdp0.as<double>(), &f->bh,
                       true, c->rec_a, c->part, grad_dev, c->scal.as<double>() + 1, &bst));
  const double bwd_ms = tb.ms();
  double sse = 0.0;
  GS_CUDA_OK(cudaMemcpyAsync(&sse, c->scal.as<double>() + 1, sizeof(double), cudaMemcpyDeviceToHost,
                             c->stream));
  if (grad_host) GS_TRY(d2h(c, grad_host, grad_dev, 3 * n));
  GS_TRY(sync(c));
  if (report) {
    report->energy = energy;
    report->residual_sse = sse;
    report->attachment = cfg->lambda * sse;
    report->total = report->energy + report->attachment;
  }
  if (stats) {
    *stats = f->stats;
    GS_TRY(flow_bh_stats(f, stats));
    stats->direct_interactions += bst.direct_interactions;
    stats->approximated_interactions += bst.approximated_interactions;
    stats->nodes_visited += bst.nodes_visited;
    stats->traversal_queries += bst.traversal_queries;
    // the energy-gradient term reuses the step-0 forward RHS (one more RHS in the reference)
    stats->forward_ms = fwd_ms - f->stats.tree_build_ms;
    stats->backward_ms = bwd_ms;
  }
  return GS_OK;
}

int evaluate_resident(gs_ctx* c, const gs_config* cfg, int64_t n, const double* q0_dev,
                      const double* box, const double* p0_dev, const double* target_dev,
                      gs_report* report, double* grad_dev, gs_stats* stats) {
  TimerInstall install(c->timer);
  return evaluate_impl(c, cfg, n, q0_dev, p0_dev, target_dev, true, box, report, nullptr, grad_dev,
                       stats);
}

bool context_is_multi(const gs_ctx* c) { return is_multi(c); }
cudaStream_t context_stream(const gs_ctx* c) { return c->stream; }

void host_box(const double* q, int64_t n, double* box) { bbox_center(q, n, box, box + 3); }

}  // namespace gsb

extern "C" {

gs_status gs_evaluate(gs_ctx* c, const gs_config* cfg, int64_t n, const double* q0,
                      const double* p0, const double* target, gs_report* report,
                      double* grad_out, gs_stats* stats) {
  if (!c || !cfg || !q0 || !p0 || !target) return bad_arg("null argument");
  TimerInstall install(c->timer);
  if (cfg->integrator != GS_EULER) return bad_arg("evaluate: the adjoint is the transpose of Euler");
  GS_TRY(gs_validate_config(cfg, nullptr));
  GS_TRY(check_n(n));
  if (is_multi(c)) return (gs_status)multi_evaluate(c, cfg, n, q0, p0, target, report, grad_out, stats);
  return (gs_status)evaluate_impl(c, cfg, n, q0, p0, target, false, nullptr, report, grad_out,
                                  nullptr, stats);
}

gs_status gs_objective(gs_ctx* c, const gs_config* cfg, int64_t n, const double* q0,
                       const double* p0, const double* target, gs_report* report) {
  if (!c || !cfg || !q0 || !p0 || !target || !report) return bad_arg("null argument");
  GS_TRY(gs_validate_config(cfg, nullptr));
  GS_TRY(check_n(n));
  std::vector<double> fq((size_t)3 * n);
  double energy = 0.0;
  GS_TRY(gs_shoot_forward(c, cfg, n, q0, p0, nullptr, nullptr, fq.data(), nullptr, &energy,
                          nullptr));
  double sse = 0.0;  // make_report, shooting.cpp:126-138 (O(N) on the host copy)
  for (int64_t i = 0; i < n; ++i) {
    const double dx = fq[3 * i] - target[3 * i], dy = fq[3 * i + 1] - target[3 * i + 1],
                 dz = fq[3 * i + 2] - target[3 * i + 2];
    sse += dx * dx + dy * dy + dz * dz;
  }
  report->energy = energy;
  report->residual_sse = sse;
  report->attachment = cfg->lambda * sse;
  report->total = report->energy + report->attachment;
  return GS_OK;
}

gs_status gs_backward_gradient(gs_ctx* c, const gs_config* cfg, int64_t n, int32_t states,
                               const double* traj_q, const double* traj_p, const double* target,
                               double* grad_out) {
  if (!c || !cfg || !traj_q || !traj_p || !target || !grad_out) return bad_arg("null argument");
  GS_TRY(gs_validate_config(cfg, nullptr));
  GS_TRY(check_n(n));
  const int T = cfg->timesteps;
  if (states != T + 1) {
    g_err = "backward_gradient: trajectory length != timesteps + 1";
    return GS_CONFIG_MISMATCH;
  }
  const int prec = cfg->precision == GS_F32 ? kF32 : kF64;
  double c0[3], ext[3];
  bbox_center(traj_q, n, c0, ext);
  const KernelConsts kc = with_ext(make_consts(cfg->sigma, prec == kF32 ? c0 : nullptr), ext);
  const size_t rb = 2 * vec_bytes(prec) * n;
  gs_flow* f = scratch_flow(c);
  GS_TRY(flow_init(f, c, cfg, n));
  DBuf& traj = c->rec_b;
  GS_TRY(traj.ensure(rb * (T + 1)));
  for (int k = 0; k <= T; ++k) {
    DBuf tmp;
    GS_TRY(upload_records(c, prec, traj_q + (size_t)3 * n * k, traj_p + (size_t)3 * n * k, n,
                          c->rec_a));
    GS_CUDA_OK(cudaMemcpyAsync(traj.as<char>() + (size_t)k * rb, c->rec_a.ptr, rb,
                               cudaMemcpyDeviceToDevice, c->stream));
  }
  GS_TRY(h2d(c, c->stage_c, target, n));
  // dH/dp(q0, p0) for the energy term (shooting.cpp:217-234)
  GS_TRY(f->dhdp0.ensure(sizeof(double) * 3 * n));
  {
    FwdEpi e;
    e.rec = traj.ptr;
    e.update = 0;
    e.dhdp_out = f->dhdp0.as<double>();
    if (cfg->backend == GS_EXACT) {
      GS_TRY(exact_stage(c->dev, prec, kc, traj.ptr, n, 0, n, f->part, e, c->stream, nullptr,
                         nullptr));
    } else {
      int blocks = 0;
      int64_t l = 0;
      GS_TRY(bh_forward_stage(c->dev, prec, kc, *cfg, traj.ptr, n, 0, n, f->bh, e, c->stream, &l,
                              &blocks, nullptr));
    }
  }
  GS_TRY(c->stage_d.ensure(sizeof(double) * 3 * n));
  GS_TRY(backward_pass(c, cfg, prec, kc, n, traj.as<char>(), rb, c->stage_c.as<double>(),
                       f->dhdp0.as<double>(), &f->bh, false, c->rec_a, c->part,
                       c->stage_d.as<double>(), nullptr, nullptr));
  GS_TRY(d2h(c, grad_out, c->stage_d.ptr, 3 * n));
  GS_TRY(sync(c));
  return GS_OK;
}

gs_status gs_warp_points(gs_ctx* c, const gs_config* cfg, int64_t n, int32_t states,
                         const double* traj_q, const double* traj_p, int64_t m, const double* x,
                         double* y_out) {
  if (!c || !cfg || !traj_q || !traj_p || !x || !y_out) return bad_arg("null argument");
  GS_TRY(gs_validate_config(cfg, nullptr));
  GS_TRY(check_n(n));
  GS_TRY(check_n(m));
  const int T = cfg->timesteps;
  if (states != T + 1) {
    g_err = "warp_points: trajectory length != timesteps + 1";
    return GS_CONFIG_MISMATCH;
  }
  const int prec = cfg->precision == GS_F32 ? kF32 : kF64;
  double c0[3], ext[3];
  bbox_center(traj_q, n, c0, ext);
  const KernelConsts kc = with_ext(make_consts(cfg->sigma, prec == kF32 ? c0 : nullptr), ext);
  const size_t rb = 2 * vec_bytes(prec) * n;
  DBuf& traj = c->rec_b;
  GS_TRY(traj.ensure(rb * T));
  for (int k = 0; k < T; ++k) {
    GS_TRY(upload_records(c, prec, traj_q + (size_t)3 * n * k, traj_p + (size_t)3 * n * k, n,
                          c->rec_a));
    GS_CUDA_OK(cudaMemcpyAsync(traj.as<char>() + (size_t)k * rb, c->rec_a.ptr, rb,
                               cudaMemcpyDeviceToDevice, c->stream));
  }
  DBuf ev;
  GS_TRY(upload_records(c, prec, x, nullptr, m, ev));
  GS_TRY(c->scal.ensure(64));
  int* bad = c->scal.as<int>() + 4;
  GS_CUDA_OK(cudaMemsetAsync(bad, 0x7f, sizeof(int), c->stream));
  gs_flow* f = scratch_flow(c);
  for (int k = 0; k < T; ++k) {
    const void* rk = traj.as<char>() + (size_t)k * rb;
    VelEpi e;
    e.m = (int)m;
    e.ev = ev.ptr;
    e.scale = 2.0;  // flow_velocity_factor, kernel_exact.hpp:28
    e.dt = 1.0 / T;
    e.update = 1;
    e.bad_step = bad;
    e.step = k + 1;
    if (cfg->backend == GS_EXACT) {
      GS_TRY(c->part.ensure((size_t)kMaxChunks * vec_bytes(prec) * m));
      const int S = vel_partials(c->dev, prec, rk, (int)n, ev.ptr, (int)m, kc, c->part.ptr,
                                 kMaxChunks, c->stream);
      if (S < 0) return (gs_status)GS_INTERNAL;
      GS_CUDA_OK(cudaGetLastError());
      e.S = S;
      e.part = c->part.ptr;
      GS_TRY(vel_epilogue(prec, e, c->stream));
    } else {
      GS_TRY(bh_velocity_step(c->dev, prec, kc, *cfg, rk, n, ev.ptr, m, f->bh, e, c->stream));
    }
  }
  int hbad = 0;
  GS_CUDA_OK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  GS_TRY(c->stage_a.ensure(sizeof(double) * 3 * m));
  GS_TRY(unpack_records(prec, ev.ptr, m, c->stage_a.as<double>(), nullptr, c->stream));
  GS_TRY(d2h(c, y_out, c->stage_a.ptr, 3 * m));
  GS_TRY(sync(c));
  if (hbad != 0x7f7f7f7f) {
    g_nonfinite = hbad;
    g_err = "non-finite state at timestep " + std::to_string(hbad);
    return GS_NONFINITE;
  }
  return GS_OK;
}

}  // extern "C"

// ----------------------------------------------------------------------------
// octree + bh_kernel entry points
// ----------------------------------------------------------------------------
struct gs_tree {
  gs_ctx* ctx = nullptr;
  int prec = kF64;
  DevTree t;
  DBuf rec;        // the build's records (index order)
  DBuf adj;        // last annotation (index order)
  DBuf part, outs, pq, stats;
  DBuf qrec, qadj;  // external queries of gs_bh_point_* (records (x, px) / (alpha_i, beta_i))
  double c0[3] = {0, 0, 0};
  double ext[3] = {0, 0, 0};  // host bounding-box extent: the walk's regime (bh_tasks)
  double sigma = -1.0;  // sigma the interaction coordinates are scaled for
  int64_t last_queries = 0;
};

static void detach_trees(gs_ctx* c) {
  for (gs_tree* t : c->trees) t->ctx = nullptr;
}

namespace {

int tree_for_sigma(gs_tree* tr, double sigma) {
  if (tr->prec == kF32 && sigma != tr->sigma) {
    const KernelConsts kc = make_consts(sigma, tr->c0);
    GS_TRY(tree_rescale(tr->prec, tr->t, tr->rec.ptr, kc, tr->ctx->stream));
  }
  tr->sigma = sigma;
  tr->t.kc = with_ext(make_consts(sigma, tr->prec == kF32 ? tr->c0 : nullptr), tr->ext);
  return GS_OK;
}

// Node windows and regime of a tree-level walk: the same choice a flow's
// stage makes (bh_tasks), so these calls exercise the production walks.
int tree_tasks(gs_tree* tr, int64_t nq, double thr, BhQuery& q) {
  int dense = 0;
  q.ntask = bh_tasks(nq, tr->t.n, thr, tr->t.kc, &dense);
  q.dense = dense;
  return q.ntask;
}

int fill_stats(gs_tree* tr, gs_stats* stats, int64_t queries) {
  if (!stats) return GS_OK;
  unsigned long long v[3] = {0, 0, 0};
  GS_CUDA_OK(cudaMemcpyAsync(v, tr->stats.ptr, sizeof v, cudaMemcpyDeviceToHost, tr->ctx->stream));
  GS_TRY(sync(tr->ctx));
  *stats = gs_stats{};
  stats->direct_interactions = v[0];
  stats->approximated_interactions = v[1];
  stats->nodes_visited = v[2];
  stats->traversal_queries = (uint64_t)queries;
  return GS_OK;
}

// RHS traversal over all tree points -> dH/dp, dH/dq (device doubles) and optionally H
int tree_rhs(gs_tree* tr, double sigma, double thr, double* dhdp_dev, double* dhdq_dev,
             double* energy_part, int* blocks, int* windows = nullptr) {
  gs_ctx* c = tr->ctx;
  const int64_t n = tr->t.n;
  GS_TRY(tree_for_sigma(tr, sigma));
  BhQuery q;
  const int K = tree_tasks(tr, n, thr, q);
  if (windows) *windows = K;
  GS_TRY(tr->part.ensure(2 * vec_bytes(tr->prec) * n * K));
  GS_TRY(tr->stats.ensure(64));
  GS_TRY(tr->pq.ensure(sizeof(uint32_t) * 3 * n));
  GS_CUDA_OK(cudaMemsetAsync(tr->stats.ptr, 0, 64, c->stream));
  q.mode = kBhRhs;
  q.tgt_begin = 0;
  q.n_tgt = (int)n;
  q.part = tr->part.ptr;
  q.per_query = tr->pq.as<uint32_t>();
  q.totals = tr->stats.as<unsigned long long>();
  q.lmd = c->lmd;
  GS_TRY(bh_traverse(c->dev, tr->prec, tr->t, sigma, thr, q, c->stream));
  FwdEpi e;
  e.rec = tr->rec.ptr;
  e.update = 0;
  e.S = K;
  e.part = tr->part.ptr;
  e.n_tgt = (int)n;
  e.cp = 2.0;
  e.cq = fwd_cq(tr->prec, tr->t.kc);
  e.dhdp_out = dhdp_dev;
  e.dhdq_out = dhdq_dev;
  e.energy_part = energy_part;
  GS_TRY(fwd_epilogue(tr->prec, e, c->stream, blocks));
  tr->last_queries = n;
  return GS_OK;
}

}  // namespace

extern "C" {

gs_status gs_tree_build(gs_ctx* c, int32_t precision, int64_t n, const double* q, const double* p,
                        gs_tree** out) {
  if (!c || !q || !p || !out) return bad_arg("null argument");
  GS_TRY(check_n(n));
  auto* tr = new gs_tree;
  tr->ctx = c;
  tr->prec = precision == GS_F32 ? kF32 : kF64;
  bbox_center(q, n, tr->c0, tr->ext);
  int s = upload_records(c, tr->prec, q, p, n, tr->rec);
  if (s == GS_OK) {
    const KernelConsts kc = make_consts(1.0, tr->prec == kF32 ? tr->c0 : nullptr);
    tr->sigma = 1.0;
    s = tree_build(c->dev, tr->prec, kc, tr->rec.ptr, n, tr->t, c->stream);
  }
  if (s == GS_OK) s = sync(c);
  if (s != GS_OK) {
    delete tr;
    return (gs_status)s;
  }
  c->trees.insert(tr);
  *out = tr;
  return GS_OK;
}

gs_status gs_tree_build_in_cell(gs_ctx* c, int32_t precision, int64_t n, const double* q,
                                const double* p, const double* cell_min, const double* cell_max,
                                gs_tree** out) {
  if (!c || !q || !p || !cell_min || !cell_max || !out) return bad_arg("null argument");
  GS_TRY(check_n(n));
  for (int64_t i = 0; i < n; ++i)  // Octree::insert, octree.cpp:76-78
    for (int a = 0; a < 3; ++a)
      if (!(q[3 * i + a] >= cell_min[a] && q[3 * i + a] <= cell_max[a])) {
        g_err = "Octree::insert: point outside the root cell";
        return GS_OUT_OF_BOUNDS;
      }
  auto* tr = new gs_tree;
  tr->ctx = c;
  tr->prec = precision == GS_F32 ? kF32 : kF64;
  bbox_center(q, n, tr->c0, tr->ext);
  const double box[6] = {cell_min[0], cell_min[1], cell_min[2], cell_max[0], cell_max[1], cell_max[2]};
  int s = upload_records(c, tr->prec, q, p, n, tr->rec);
  if (s == GS_OK) {
    const KernelConsts kc = make_consts(1.0, tr->prec == kF32 ? tr->c0 : nullptr);
    tr->sigma = 1.0;
    s = tree_build(c->dev, tr->prec, kc, tr->rec.ptr, n, tr->t, c->stream, box);
  }
  if (s == GS_OK) s = sync(c);
  if (s != GS_OK) {
    delete tr;
    return (gs_status)s;
  }
  c->trees.insert(tr);
  *out = tr;
  return GS_OK;
}

void gs_tree_free(gs_tree* tr) {
  if (!tr) return;
  if (tr->ctx) {
    cudaStreamSynchronize(tr->ctx->stream);
    tr->ctx->trees.erase(tr);
  }
  delete tr;
}

int64_t gs_tree_node_count(const gs_tree* tr) {
  return tr ? tree_node_count(const_cast<gs_tree*>(tr)->t, tr->ctx->stream) : 0;
}
int64_t gs_tree_point_count(const gs_tree* tr) { return tr ? tr->t.n : 0; }

gs_status gs_tree_accumulate_adjoints(gs_tree* tr, const double* alpha, const double* beta) {
  if (!tr || !alpha || !beta) return bad_arg("null argument");
  GS_TRY(upload_records(tr->ctx, tr->prec, alpha, beta, tr->t.n, tr->adj));
  GS_TRY(tree_accumulate(tr->prec, tr->t, tr->adj.ptr, tr->ctx->stream));
  return (gs_status)sync(tr->ctx);
}

gs_status gs_tree_download(const gs_tree* tr, int32_t* order, uint64_t* key_hi, uint64_t* key_lo,
                           int32_t* level, int32_t* parent, int32_t* skip, int32_t* range,
                           double* boxes, double* sums, uint32_t* count) {
  if (!tr) return bad_arg("null tree");
  return (gs_status)tree_download(const_cast<gs_tree*>(tr)->t, tr->ctx->stream, order, key_hi, key_lo, level, parent,
                                  skip, range, boxes, sums, count);
}

gs_status gs_bh_rhs(gs_tree* tr, double sigma, double thr, double* dHdp, double* dHdq,
                    gs_stats* stats) {
  if (!tr) return bad_arg("null tree");
  gs_ctx* c = tr->ctx;
  const int64_t n = tr->t.n;
  GS_TRY(tr->outs.ensure(sizeof(double) * 6 * n));
  double* dp = tr->outs.as<double>();
  GS_TRY(tree_rhs(tr, sigma, thr, dp, dp + 3 * n, nullptr, nullptr));
  GS_TRY(d2h(c, dHdp, dp, 3 * n));
  GS_TRY(d2h(c, dHdq, dp + 3 * n, 3 * n));
  GS_TRY(sync(c));
  return (gs_status)fill_stats(tr, stats, n);
}

gs_status gs_bh_hamiltonian(gs_tree* tr, double sigma, double thr, double* h_out, gs_stats* stats) {
  if (!tr || !h_out) return bad_arg("null argument");
  gs_ctx* c = tr->ctx;
  const int64_t n = tr->t.n;
  GS_TRY(c->epart.ensure(sizeof(double) * (n / 128 + 8)));
  GS_TRY(c->scal.ensure(64));
  int blocks = 0, K = 1;
  GS_TRY(c->epart.ensure(sizeof(double) * (n * 64 / 128 + 8)));
  GS_TRY(tree_rhs(tr, sigma, thr, nullptr, nullptr, c->epart.as<double>(), &blocks, &K));
  if (c->lmd)  // the dot is scaled too (bh_kernel.cpp:184): the per-target sums of c over all
               // K node windows' partials ([K][n][2], B.w)
    GS_TRY(sum_part_w(tr->prec, tr->part.ptr, (int)(n * K), 2, 1, c->epart.as<double>(), &blocks,
                      c->stream));
  GS_TRY(reduce_sum(c->epart.as<double>(), blocks, c->scal.as<double>(), c->stream));
  double h = 0.0;
  GS_CUDA_OK(cudaMemcpyAsync(&h, c->scal.ptr, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  GS_TRY(sync(c));
  // bh_hamiltonian = sum_j p_j . sum_units G P = 1/2 <p, dH/dp> (bh_kernel.cpp:162-191);
  // under literal-mean-dot, sum_j sum_units (p_j . P) scale G directly
  *h_out = c->lmd ? h : 0.5 * h;
  return (gs_status)fill_stats(tr, stats, n);
}

gs_status gs_bh_velocity(gs_tree* tr, int64_t m, const double* x, double sigma, double thr,
                         double* v_out, gs_stats* stats) {
  if (!tr || !x || !v_out) return bad_arg("null argument");
  GS_TRY(check_n(m));
  gs_ctx* c = tr->ctx;
  GS_TRY(tree_for_sigma(tr, sigma));
  GS_TRY(upload_records(c, tr->prec, x, nullptr, m, tr->qrec));
  BhQuery q;
  const int K = tree_tasks(tr, m, thr, q);
  GS_TRY(tr->part.ensure(vec_bytes(tr->prec) * m * K));
  GS_TRY(tr->stats.ensure(64));
  GS_TRY(tr->pq.ensure(sizeof(uint32_t) * 3 * m));
  GS_TRY(tr->outs.ensure(sizeof(double) * 3 * m));
  GS_CUDA_OK(cudaMemsetAsync(tr->stats.ptr, 0, 64, c->stream));
  q.mode = kBhVel;
  q.ev = tr->qrec.ptr;
  q.m = (int)m;
  q.part = tr->part.ptr;
  q.per_query = tr->pq.as<uint32_t>();
  q.totals = tr->stats.as<unsigned long long>();
  GS_TRY(bh_traverse(c->dev, tr->prec, tr->t, sigma, thr, q, c->stream));
  VelEpi e;
  e.m = (int)m;
  e.S = K;
  e.part = tr->part.ptr;
  e.scale = 1.0;
  e.v_out = tr->outs.as<double>();
  GS_TRY(vel_epilogue(tr->prec, e, c->stream));
  GS_TRY(d2h(c, v_out, tr->outs.ptr, 3 * m));
  GS_TRY(sync(c));
  tr->last_queries = m;
  return (gs_status)fill_stats(tr, stats, m);
}

gs_status gs_bh_query_stats(const gs_tree* tr, uint64_t* per_query) {
  if (!tr || !per_query) return bad_arg("null argument");
  std::vector<uint32_t> v((size_t)3 * tr->last_queries);
  if (!v.empty()) {
    GS_CUDA_OK(cudaMemcpyAsync(v.data(), tr->pq.ptr, sizeof(uint32_t) * v.size(),
                               cudaMemcpyDeviceToHost, tr->ctx->stream));
    GS_TRY(sync(tr->ctx));
  }
  for (size_t i = 0; i < v.size(); ++i) per_query[i] = v[i];
  return GS_OK;
}

gs_status gs_bh_hessian_products(gs_tree* tr, const double* alpha, const double* beta,
                                 double sigma, double thr, double* pq, double* pp, double* qq,
                                 double* qp, gs_stats* stats) {
  if (!tr || !alpha || !beta) return bad_arg("null argument");
  gs_ctx* c = tr->ctx;
  const int64_t n = tr->t.n;
  GS_TRY(tree_for_sigma(tr, sigma));
  DBuf adj;
  GS_TRY(upload_records(c, tr->prec, alpha, beta, n, adj));
  if (!tr->t.adj_valid) GS_TRY(tree_accumulate(tr->prec, tr->t, adj.ptr, c->stream));
  else GS_TRY(tree_set_point_adjoints(tr->prec, tr->t, adj.ptr, c->stream));
  BhQuery q;
  const int K = tree_tasks(tr, n, thr, q);
  GS_TRY(tr->part.ensure(4 * vec_bytes(tr->prec) * n * K));
  GS_TRY(tr->stats.ensure(64));
  GS_TRY(tr->pq.ensure(sizeof(uint32_t) * 3 * n));
  GS_TRY(tr->outs.ensure(sizeof(double) * 12 * n));
  GS_CUDA_OK(cudaMemsetAsync(tr->stats.ptr, 0, 64, c->stream));
  q.mode = kBhHess;
  q.tgt_begin = 0;
  q.n_tgt = (int)n;
  q.part = tr->part.ptr;
  q.per_query = tr->pq.as<uint32_t>();
  q.totals = tr->stats.as<unsigned long long>();
  q.lmd = c->lmd;
  GS_TRY(bh_traverse(c->dev, tr->prec, tr->t, sigma, thr, q, c->stream));
  const KernelConsts& kc = tr->t.kc;
  const double cd = tr->prec == kF32 ? kc.two_over_s / kc.kappa : kc.two_over_s;
  BwdEpi e;
  e.n_tgt = (int)n;
  e.S = K;
  e.part = tr->part.ptr;
  e.update = 0;
  e.cpq = -cd;
  e.cpp = 2.0;
  e.cqq = kc.two_over_s;
  e.cqp = -cd;
  double* o = tr->outs.as<double>();
  for (int k = 0; k < 4; ++k) e.out[k] = o + (size_t)3 * n * k;
  GS_TRY(bwd_epilogue(tr->prec, e, c->stream));
  double* hs[4] = {pq, pp, qq, qp};
  for (int k = 0; k < 4; ++k) GS_TRY(d2h(c, hs[k], o + (size_t)3 * n * k, 3 * n));
  GS_TRY(sync(c));
  tr->last_queries = n;
  return (gs_status)fill_stats(tr, stats, n);
}

gs_status gs_bh_point_gradients(gs_tree* tr, int64_t m, const double* x, const double* px,
                                double sigma, double thr, double* dHdp, double* dHdq,
                                gs_stats* stats) {
  if (!tr || !x || !px) return bad_arg("null argument");
  GS_TRY(check_n(m));
  gs_ctx* c = tr->ctx;
  GS_TRY(tree_for_sigma(tr, sigma));
  GS_TRY(upload_records(c, tr->prec, x, px, m, tr->qrec));
  BhQuery q;
  const int K = tree_tasks(tr, m, thr, q);
  GS_TRY(tr->part.ensure(2 * vec_bytes(tr->prec) * m * K));
  GS_TRY(tr->stats.ensure(64));
  GS_TRY(tr->pq.ensure(sizeof(uint32_t) * 3 * m));
  GS_TRY(tr->outs.ensure(sizeof(double) * 6 * m));
  GS_CUDA_OK(cudaMemsetAsync(tr->stats.ptr, 0, 64, c->stream));
  q.mode = kBhRhs;
  q.by_index = 1;  // external (x, px) records, not the tree's points
  q.ev = tr->qrec.ptr;
  q.tgt_begin = 0;
  q.n_tgt = (int)m;
  q.part = tr->part.ptr;
  q.per_query = tr->pq.as<uint32_t>();
  q.totals = tr->stats.as<unsigned long long>();
  q.lmd = c->lmd;
  GS_TRY(bh_traverse(c->dev, tr->prec, tr->t, sigma, thr, q, c->stream));
  double* o = tr->outs.as<double>();
  FwdEpi e;
  e.rec = tr->qrec.ptr;
  e.update = 0;
  e.S = K;
  e.part = tr->part.ptr;
  e.n_tgt = (int)m;
  e.cp = 2.0;
  e.cq = fwd_cq(tr->prec, tr->t.kc);
  e.dhdp_out = o;
  e.dhdq_out = o + 3 * m;
  GS_TRY(fwd_epilogue(tr->prec, e, c->stream, nullptr));
  GS_TRY(d2h(c, dHdp, o, 3 * m));
  GS_TRY(d2h(c, dHdq, o + 3 * m, 3 * m));
  GS_TRY(sync(c));
  tr->last_queries = m;
  return (gs_status)fill_stats(tr, stats, m);
}

gs_status gs_bh_point_hessian_products(gs_tree* tr, int64_t m, const double* qi, const double* pi,
                                       const double* alpha_i, const double* beta_i,
                                       const double* alpha, const double* beta, double sigma,
                                       double thr, double* pq, double* pp, double* qq, double* qp,
                                       gs_stats* stats) {
  if (!tr || !qi || !pi || !alpha_i || !beta_i) return bad_arg("null argument");
  if (!alpha != !beta) return bad_arg("alpha and beta must both be given or both be NULL");
  GS_TRY(check_n(m));
  gs_ctx* c = tr->ctx;
  const int64_t n = tr->t.n;
  GS_TRY(tree_for_sigma(tr, sigma));
  if (!tr->t.adj_valid) {  // never annotated: the reference's node sums are zero (Node defaults)
    GS_TRY(tr->adj.ensure(2 * vec_bytes(tr->prec) * n));
    GS_CUDA_OK(cudaMemsetAsync(tr->adj.ptr, 0, 2 * vec_bytes(tr->prec) * n, c->stream));
    GS_TRY(tree_accumulate(tr->prec, tr->t, tr->adj.ptr, c->stream));
  }
  if (alpha) {  // direct terms read these per-point adjoints; node sums stay as annotated
    DBuf adj;
    GS_TRY(upload_records(c, tr->prec, alpha, beta, n, adj));
    GS_TRY(tree_set_point_adjoints(tr->prec, tr->t, adj.ptr, c->stream));
  }
  GS_TRY(upload_records(c, tr->prec, qi, pi, m, tr->qrec));
  GS_TRY(upload_records(c, tr->prec, alpha_i, beta_i, m, tr->qadj));
  BhQuery q;
  const int K = tree_tasks(tr, m, thr, q);
  GS_TRY(tr->part.ensure(4 * vec_bytes(tr->prec) * m * K));
  GS_TRY(tr->stats.ensure(64));
  GS_TRY(tr->pq.ensure(sizeof(uint32_t) * 3 * m));
  GS_TRY(tr->outs.ensure(sizeof(double) * 12 * m));
  GS_CUDA_OK(cudaMemsetAsync(tr->stats.ptr, 0, 64, c->stream));
  q.mode = kBhHess;
  q.by_index = 1;
  q.ev = tr->qrec.ptr;
  q.eadj = tr->qadj.ptr;
  q.tgt_begin = 0;
  q.n_tgt = (int)m;
  q.part = tr->part.ptr;
  q.per_query = tr->pq.as<uint32_t>();
  q.totals = tr->stats.as<unsigned long long>();
  q.lmd = c->lmd;
  GS_TRY(bh_traverse(c->dev, tr->prec, tr->t, sigma, thr, q, c->stream));
  const KernelConsts& kc = tr->t.kc;
  const double cd = tr->prec == kF32 ? kc.two_over_s / kc.kappa : kc.two_over_s;
  BwdEpi e;
  e.n_tgt = (int)m;
  e.S = K;
  e.part = tr->part.ptr;
  e.update = 0;
  e.cpq = -cd;
  e.cpp = 2.0;
  e.cqq = kc.two_over_s;
  e.cqp = -cd;
  double* o = tr->outs.as<double>();
  for (int k = 0; k < 4; ++k) e.out[k] = o + (size_t)3 * m * k;
  GS_TRY(bwd_epilogue(tr->prec, e, c->stream));
  double* hs[4] = {pq, pp, qq, qp};
  for (int k = 0; k < 4; ++k) GS_TRY(d2h(c, hs[k], o + (size_t)3 * m * k, 3 * m));
  GS_TRY(sync(c));
  tr->last_queries = m;
  return (gs_status)fill_stats(tr, stats, m);
}

}  // extern "C"

// ----------------------------------------------------------------------------
// Multi-device contexts: one process drives G devices. Target
// points are cut into G contiguous shards (Barnes-Hut: of the Morton-ordered
// records, so a shard is a compact region). Every device holds all n records
// and computes its shard's RHS against all of them; the stage epilogue stores
// the shard's updated records into its own next buffer AND into every peer's
// (P2P stores over NVLink / NVSwitch: the all-gather is fused into the
// epilogue). Buffers ping-pong per stage, so a peer never overwrites records
// a device is still reading; one event wait per peer and stage orders them.
// The adjoint pass does the same with the (alpha, beta) records. Exact RHS
// shards are planned as the full problem (rhs_partials plan_tgt), so their
// partial sums -- and the flow -- are bit-identical to one device's.
// ----------------------------------------------------------------------------
namespace {

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int d) {
    cudaGetDevice(&prev);
    cudaSetDevice(d);
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

void shard_of(int64_t n, int G, int d, int64_t* b, int64_t* cnt) {
  const int64_t base = n / G, extra = n % G;
  *b = d * base + std::min<int64_t>(d, extra);
  *cnt = base + (d < extra ? 1 : 0);
}

int sub_dev(const gs_flow* s) { return s->ctx->dev.id; }

// every shard's stream waits for every other shard's last recorded event
int multi_wait_all(gs_ctx* c) {
  const int G = (int)c->subs.size();
  for (int d = 0; d < G; ++d) {
    DevGuard g(c->subs[d]->dev.id);
    for (int o = 0; o < G; ++o)
      if (o != d) GS_CUDA_OK(cudaStreamWaitEvent(c->subs[d]->stream, c->ev[o], 0));
  }
  return GS_OK;
}

int multi_record(gs_ctx* c, int d) {
  GS_CUDA_OK(cudaEventRecord(c->ev[d], c->subs[d]->stream));
  return GS_OK;
}

// The peers' copies of a shard written by shard d: P2P stores from the
// epilogue (peer_stores), else explicit peer copies after it.
PeerOut peer_bufs(gs_ctx* c, const std::vector<void*>& bufs, int d) {
  PeerOut po;
  if (!c->peer_stores) return po;
  for (int o = 0; o < (int)bufs.size(); ++o)
    if (o != d) po.buf[po.n++] = bufs[o];
  return po;
}

int peer_copies(gs_ctx* c, const std::vector<void*>& bufs, int d, size_t off, size_t bytes) {
  if (c->peer_stores || bytes == 0) return GS_OK;
  for (int o = 0; o < (int)bufs.size(); ++o)
    if (o != d)
      GS_CUDA_OK(cudaMemcpyPeerAsync(static_cast<char*>(bufs[o]) + off, c->subs[o]->dev.id,
                                     static_cast<char*>(bufs[d]) + off, c->subs[d]->dev.id, bytes,
                                     c->subs[d]->stream));
  return GS_OK;
}

int multi_flow_init(gs_flow* f, gs_ctx* c, const gs_config* cfg, int64_t n) {
  const int G = (int)c->subs.size();
  f->ctx = c;
  f->cfg = *cfg;
  f->prec = cfg->precision == GS_F32 ? kF32 : kF64;
  f->n = n;
  f->shard_begin = 0;
  f->shard_count = n;
  f->steps_done = 0;
  while ((int)f->subs.size() < G) f->subs.push_back(new gs_flow);
  for (int d = 0; d < G; ++d) {
    DevGuard g(c->subs[d]->dev.id);
    gs_flow* s = f->subs[d];
    GS_TRY(flow_init(s, c->subs[d], cfg, n));
    shard_of(n, G, d, &s->shard_begin, &s->shard_count);
    s->plan_tgt = (int)n;  // bit-identical partial sums to the unsharded RHS
    GS_TRY(s->rec_next.ensure(2 * vec_bytes(s->prec) * n));
  }
  return GS_OK;
}

int multi_flow_upload(gs_flow* f, const double* q0, const double* p0) {
  gs_ctx* c = f->ctx;
  GS_TRY(multi_wait_all(c));  // nothing may still write into the buffers
  for (int d = 0; d < (int)f->subs.size(); ++d) {
    gs_flow* s = f->subs[d];
    DevGuard g(sub_dev(s));
    GS_TRY(flow_upload(s, q0, p0));
    if (s->cfg.backend == GS_BARNES_HUT && f->subs.size() > 1) GS_TRY(flow_morton_permute(s));
    GS_TRY(multi_record(c, d));
  }
  f->steps_done = 0;
  return GS_OK;
}

// One symmetric exact stage across the devices (pair rows):
// every device evaluates its rows of the tile-pair grid and folds them per
// target; each shard then peer-copies the G partials of its targets (device
// order) and runs its epilogue over them, storing its records into every
// peer's next buffer as in the gather path.
int multi_pair_stage(gs_flow* f, int stage, const std::vector<void*>& next) {
  gs_ctx* c = f->ctx;
  const int G = (int)f->subs.size();
  const int n = (int)f->n;
  const size_t rb = 2 * vec_bytes(f->prec), pb = 2 * sizeof(float4);
  GS_TRY(multi_wait_all(c));
  for (int d = 0; d < G; ++d) {
    gs_flow* s = f->subs[d];
    DevGuard g(sub_dev(s));
    GS_TRY(s->part.ensure(sym_part_bytes(n)));
    GS_TRY(s->pair_out.ensure(pb * n));
    GS_TRY(s->pair_in.ensure(pb * G * std::max<int64_t>(s->shard_count, 1)));
    TimerInstall install(s->timer);
    kt_mark(0, s->ctx->stream);
    rhs_sym_rows(s->rec.ptr, n, s->kc, s->part.ptr, s->pair_out.ptr, d, G, s->ctx->stream);
    kt_mark(0, s->ctx->stream);
    GS_CUDA_OK(cudaGetLastError());
    s->launches += 2;
    GS_TRY(multi_record(c, d));
  }
  GS_TRY(multi_wait_all(c));
  for (int d = 0; d < G; ++d) {
    gs_flow* s = f->subs[d];
    DevGuard g(sub_dev(s));
    cudaStream_t st = s->ctx->stream;
    for (int o = 0; o < G; ++o)
      GS_CUDA_OK(cudaMemcpyPeerAsync(s->pair_in.as<char>() + pb * o * s->shard_count, sub_dev(s),
                                     f->subs[o]->pair_out.as<char>() + pb * s->shard_begin,
                                     sub_dev(f->subs[o]), pb * s->shard_count, st));
    FwdEpi e;
    bool first = false;
    GS_TRY(flow_epi(s, stage, s->rec.ptr, s->rec_next.ptr, e, first));
    e.peers = peer_bufs(c, next, d);
    e.S = G;
    e.part = s->pair_in.ptr;
    e.n_tgt = (int)s->shard_count;
    e.tgt_begin = (int)s->shard_begin;
    e.cp = 2.0;
    e.cq = fwd_cq(kF32, s->kc);
    int blocks = 0;
    GS_TRY(fwd_epilogue(kF32, e, st, &blocks));
    s->launches += 1;
    s->stats.direct_interactions += (uint64_t)n * (uint64_t)s->shard_count;
    s->stats.traversal_queries += (uint64_t)s->shard_count;
    if (first) {
      s->have_energy_part = true;
      s->energy_blocks = blocks;
    }
    GS_TRY(peer_copies(c, next, d, rb * s->shard_begin, rb * s->shard_count));
    GS_TRY(multi_record(c, d));
  }
  return GS_OK;
}

bool multi_pairs(const gs_flow* f) {
  return f->subs.size() > 1 && f->cfg.backend == GS_EXACT && f->prec == kF32 &&
         !(f->cfg.flags & (GS_FLAG_EXACT_CUTOFF | GS_FLAG_EXACT_MORTON)) &&
         use_sym(kF32, (int)f->n, 0, (int)f->n, -1) && !sym_grouped((int)f->n);
}

int multi_flow_advance(gs_flow* f, int steps) {
  gs_ctx* c = f->ctx;
  const int G = (int)f->subs.size();
  const size_t rb = 2 * vec_bytes(f->prec);
  const bool pairs = multi_pairs(f);
  for (int k = 0; k < steps; ++k) {
    for (int stage = 0; stage < flow_stages(f); ++stage) {
      GS_TRY(multi_wait_all(c));  // the previous stage of every shard is in every buffer
      std::vector<void*> next(G);
      for (int d = 0; d < G; ++d) next[d] = f->subs[d]->rec_next.ptr;
      if (pairs) GS_TRY(multi_pair_stage(f, stage, next));
      for (int d = 0; d < G && !pairs; ++d) {
        gs_flow* s = f->subs[d];
        DevGuard g(sub_dev(s));
        s->peers = peer_bufs(c, next, d);
        GS_TRY(flow_stage(s, stage, s->rec.ptr, s->rec_next.ptr));
        s->peers = PeerOut{};
        GS_TRY(peer_copies(c, next, d, rb * s->shard_begin, rb * s->shard_count));
        GS_TRY(multi_record(c, d));
      }
      for (gs_flow* s : f->subs) {
        std::swap(s->rec.ptr, s->rec_next.ptr);
        std::swap(s->rec.bytes, s->rec_next.bytes);
      }
    }
    for (gs_flow* s : f->subs) {
      ++s->steps_done;
    }
    ++f->steps_done;
  }
  return GS_OK;
}

int multi_flow_check(gs_flow* f) {
  int first = GS_OK;
  int step = INT32_MAX;
  for (gs_flow* s : f->subs) {
    DevGuard g(sub_dev(s));
    const int st = flow_check(s);
    if (st == GS_NONFINITE) step = std::min(step, g_nonfinite);
    if (st != GS_OK && first == GS_OK) first = st;
  }
  if (first == GS_NONFINITE) {
    g_nonfinite = step;
    g_err = "non-finite state at timestep " + std::to_string(step);
  }
  return first;
}

int multi_flow_download(gs_flow* f, double* q, double* p) {
  gs_ctx* c = f->ctx;
  GS_TRY(multi_wait_all(c));  // shard 0's buffers hold every shard once the others are done
  gs_flow* s = f->subs[0];
  DevGuard g(sub_dev(s));
  return gs_flow_download(s, q, p);
}

int multi_flow_stats(gs_flow* f, gs_stats* out) {
  *out = gs_stats{};
  for (gs_flow* s : f->subs) {
    DevGuard g(sub_dev(s));
    gs_stats t = s->stats;
    GS_TRY(flow_bh_stats(s, &t));
    out->direct_interactions += t.direct_interactions;
    out->approximated_interactions += t.approximated_interactions;
    out->nodes_visited += t.nodes_visited;
    out->traversal_queries += t.traversal_queries;
    out->tree_build_ms += t.tree_build_ms;
  }
  return GS_OK;
}

// H(q0, p0) = 1/2 <p0, dH/dp>: each shard's part, summed in shard order
int multi_flow_energy(gs_flow* f, double* out) {
  double h = 0.0;
  for (gs_flow* s : f->subs) {
    DevGuard g(sub_dev(s));
    double e = 0.0;
    GS_TRY(flow_energy(s, &e));
    h += e;
  }
  *out = h;
  return GS_OK;
}

int multi_evaluate(gs_ctx* c, const gs_config* cfg, int64_t n, const double* q0, const double* p0,
                   const double* target, gs_report* report, double* grad_out, gs_stats* stats) {
  const int T = cfg->timesteps;
  const int G = (int)c->subs.size();
  gs_flow* f = scratch_flow(c);
  GS_TRY(multi_flow_init(f, c, cfg, n));
  for (gs_flow* s : f->subs) s->want_energy = true;
  GS_TRY(multi_flow_upload(f, q0, p0));
  const int prec = f->prec;
  const size_t rb = 2 * vec_bytes(prec) * n, rec1 = 2 * vec_bytes(prec);
  const bool bh = cfg->backend == GS_BARNES_HUT;
  const bool permuted = f->subs[0]->permuted;
  const auto t0 = std::chrono::steady_clock::now();
  // per shard: trajectory traj[0..T] (all n records, sub-context rec_b), the
  // target (stage_c, in the records' order), the adjoints (rec_a / rec_next)
  std::vector<char*> traj(G);
  for (int d = 0; d < G; ++d) {
    gs_flow* s = f->subs[d];
    gs_ctx* sc = s->ctx;
    DevGuard g(sc->dev.id);
    GS_TRY(sc->rec_b.ensure(rb * (T + 1)));
    traj[d] = sc->rec_b.as<char>();
    GS_CUDA_OK(cudaMemcpyAsync(traj[d], s->rec.ptr, rb, cudaMemcpyDeviceToDevice, sc->stream));
    GS_TRY(h2d(sc, sc->stage_c, target, n));
    if (permuted) {
      GS_TRY(sc->stage_d.ensure(sizeof(double) * 3 * n));
      GS_TRY(gather_rows3(sc->stage_c.as<double>(), s->order.as<int>(), n, sc->stage_d.as<double>(),
                          sc->stream));
      std::swap(sc->stage_c.ptr, sc->stage_d.ptr);
      std::swap(sc->stage_c.bytes, sc->stage_d.bytes);
    }
    if (bh) GS_TRY(bh_keep_trees(s->bh, T));
    GS_TRY(multi_record(c, d));
  }
  // forward: step k reads traj[k], the epilogues store traj[k+1] on every device
  for (int k = 0; k < T; ++k) {
    GS_TRY(multi_wait_all(c));
    std::vector<void*> next(G);
    for (int d = 0; d < G; ++d) next[d] = traj[d] + (size_t)(k + 1) * rb;
    for (int d = 0; d < G; ++d) {
      gs_flow* s = f->subs[d];
      DevGuard g(sub_dev(s));
      s->peers = peer_bufs(c, next, d);
      s->bh.cache_slot = bh ? k : -1;
      const int st = flow_stage(s, 0, traj[d] + (size_t)k * rb, next[d]);
      s->bh.cache_slot = -1;
      s->peers = PeerOut{};
      GS_TRY(st);
      GS_TRY(peer_copies(c, next, d, rec1 * s->shard_begin, rec1 * s->shard_count));
      ++s->steps_done;
      GS_TRY(multi_record(c, d));
    }
  }
  GS_TRY(multi_flow_check(f));
  double energy = 0.0;
  GS_TRY(multi_flow_energy(f, &energy));
  const auto t1 = std::chrono::steady_clock::now();
  // backward: every device initialises the full adjoints from traj[T] (same
  // values everywhere), then each step updates its shard into every device
  std::vector<void*> acur(G), anext(G);
  double sse = 0.0;
  GS_TRY(multi_wait_all(c));
  for (int d = 0; d < G; ++d) {
    gs_flow* s = f->subs[d];
    gs_ctx* sc = s->ctx;
    DevGuard g(sc->dev.id);
    GS_TRY(sc->rec_a.ensure(rb));
    GS_TRY(sc->epart.ensure(sizeof(double) * (n / 128 + 8)));
    GS_TRY(sc->scal.ensure(64));
    acur[d] = sc->rec_a.ptr;
    anext[d] = s->rec_next.ptr;
    int blocks = 0;
    GS_TRY(adjoint_init(prec, traj[d] + (size_t)T * rb, sc->stage_c.as<double>(), cfg->lambda, n,
                        acur[d], sc->epart.as<double>(), &blocks, sc->stream));
    if (d == 0) {
      GS_TRY(reduce_sum(sc->epart.as<double>(), blocks, sc->scal.as<double>() + 1, sc->stream));
      GS_CUDA_OK(cudaMemcpyAsync(&sse, sc->scal.as<double>() + 1, sizeof(double),
                                 cudaMemcpyDeviceToHost, sc->stream));
    }
    GS_TRY(multi_record(c, d));
  }
  gs_stats bst{};
  for (int k = T - 1; k >= 0; --k) {
    GS_TRY(multi_wait_all(c));
    for (int d = 0; d < G; ++d) {
      gs_flow* s = f->subs[d];
      gs_ctx* sc = s->ctx;
      DevGuard g(sc->dev.id);
      const double cd = prec == kF32 ? s->kc.two_over_s / s->kc.kappa : s->kc.two_over_s;
      BwdEpi e;
      e.update = 1;
      e.dt = 1.0 / T;
      e.cpq = -cd;
      e.cpp = 2.0;
      e.cqq = s->kc.two_over_s;
      e.cqp = -cd;
      e.adj_out = anext[d];
      e.peers = peer_bufs(c, anext, d);
      GS_TRY(backward_step(sc, cfg, prec, s->kc, n, s->shard_begin, s->shard_count,
                           traj[d] + (size_t)k * rb, acur[d], k, &s->bh, true, sc->part, e, &bst,
                           (int)n));
      GS_TRY(peer_copies(c, anext, d, rec1 * s->shard_begin, rec1 * s->shard_count));
      GS_TRY(multi_record(c, d));
    }
    std::swap(acur, anext);
  }
  // gradient = beta_0 + dH/dp(q0, p0) per shard, back to the caller's order
  std::vector<double> g_host(permuted ? (size_t)3 * n : 0);
  double* gdst = permuted ? g_host.data() : grad_out;
  for (int d = 0; d < G; ++d) {
    gs_flow* s = f->subs[d];
    gs_ctx* sc = s->ctx;
    DevGuard g(sc->dev.id);
    GS_TRY(sc->stage_d.ensure(sizeof(double) * 3 * std::max<int64_t>(s->shard_count, 1)));
    GS_TRY(gradient_finalize(prec, static_cast<char*>(acur[d]) + rec1 * s->shard_begin,
                             s->dhdp0.as<double>(), s->shard_count, sc->stage_d.as<double>(),
                             sc->stream));
    if (gdst) GS_TRY(d2h(sc, gdst + 3 * s->shard_begin, sc->stage_d.ptr, 3 * s->shard_count));
  }
  std::vector<int32_t> order(permuted ? n : 0);
  if (permuted) {
    gs_ctx* sc = f->subs[0]->ctx;
    DevGuard g(sc->dev.id);
    GS_CUDA_OK(cudaMemcpyAsync(order.data(), f->subs[0]->order.ptr, sizeof(int32_t) * n,
                               cudaMemcpyDeviceToHost, sc->stream));
  }
  for (gs_ctx* sc : c->subs) {
    DevGuard g(sc->dev.id);
    GS_TRY(sync(sc));
  }
  if (permuted && grad_out)
    for (int64_t t = 0; t < n; ++t)
      for (int a = 0; a < 3; ++a) grad_out[3 * order[t] + a] = g_host[3 * t + a];
  const auto t2 = std::chrono::steady_clock::now();
  if (report) {
    report->energy = energy;
    report->residual_sse = sse;
    report->attachment = cfg->lambda * sse;
    report->total = report->energy + report->attachment;
  }
  if (stats) {
    GS_TRY(multi_flow_stats(f, stats));
    stats->direct_interactions += bst.direct_interactions;
    stats->approximated_interactions += bst.approximated_interactions;
    stats->nodes_visited += bst.nodes_visited;
    stats->traversal_queries += bst.traversal_queries;
    stats->forward_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    stats->backward_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
  }
  return GS_OK;
}

}  // namespace

extern "C" {

gs_ctx* gs_create_multi(int32_t count, const int32_t* devices, gs_status* status) {
  if (count < 1 || count > kMaxPeers + 1 || !devices) {
    g_err = "gs_create_multi: 1.." + std::to_string(kMaxPeers + 1) + " devices";
    if (status) *status = GS_INVALID_ARGUMENT;
    return nullptr;
  }
  gs_ctx* c = gs_create(devices[0], status);
  if (!c) return nullptr;
  for (int d = 0; d < count; ++d) {
    gs_ctx* s = gs_create(devices[d], status);
    if (!s) {
      gs_destroy(c);
      return nullptr;
    }
    c->subs.push_back(s);
    cudaEvent_t e{};
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    c->ev.push_back(e);
  }
  // P2P stores need peer access between every pair of distinct devices
  bool p2p = true;
  for (int a = 0; a < count && p2p; ++a)
    for (int b = 0; b < count && p2p; ++b) {
      if (devices[a] == devices[b]) continue;
      int ok = 0;
      cudaDeviceCanAccessPeer(&ok, devices[a], devices[b]);
      if (!ok) { p2p = false; break; }
      cudaSetDevice(devices[a]);
      const cudaError_t e = cudaDeviceEnablePeerAccess(devices[b], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) p2p = false;
      cudaGetLastError();  // clear "already enabled"
    }
  // GS_MULTI_COPIES=1: exchange by explicit peer copies instead (A/B, tests)
  if (const char* e = std::getenv("GS_MULTI_COPIES")) p2p = p2p && std::atoi(e) == 0;
  c->peer_stores = p2p;
  cudaSetDevice(devices[0]);
  if (status) *status = GS_OK;
  return c;
}

int32_t gs_ctx_device_count(const gs_ctx* c) {
  return c ? (c->subs.empty() ? 1 : (int32_t)c->subs.size()) : 0;
}

int32_t gs_ctx_peer_stores(const gs_ctx* c) { return c && !c->subs.empty() && c->peer_stores ? 1 : 0; }

}  // extern "C"
