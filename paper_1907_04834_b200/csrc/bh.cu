// bh.cu -- warp-cooperative Barnes-Hut traversal on sm_100a.
//
// Replaces traverse() + the per-query kernels of bh_kernel.cpp:30-160. Per
// query the reference walks the tree with a LIFO stack: a leaf contributes its
// point(s) directly (:40-45), a node whose tight box lies farther than the
// threshold contributes ONE term at its centroid with its aggregate momentum /
// adjoints (:46-48, :74-77, :143-157), anything else is opened (:49-57).
//
// Here the nodes are in depth-first pre-order with skip pointers, so a query's
// walk is a monotone sweep: visit n; leaf/far -> next = skip[n]; open ->
// next = n + 1. Queries are the tree's points in leaf (Morton) order, so a
// warp holds 32 neighbours. k_bh_ws (default) walks each lane independently:
// per iteration a lane visits one node (64-B record = its unit + its box,
// two 256-bit loads) or takes one point of its pending direct range, and all
// lanes holding a unit evaluate it together. A leaf, a twig (children all
// leaves) or a node whose FARTHEST box point is within the threshold -- all
// of whose descendants the reference would open down to their leaves -- is a
// contiguous range of leaf-order points; long ranges are swept by the whole
// warp. k_bh_grp walks the union of the warp's node sets and sweeps the union
// of the lanes' direct ranges with broadcast loads (dense regimes). The
// interaction set and the per-query (direct, approximated, visited) counts
// equal the reference's exactly; only the summation order differs.
//
// The gate min_distance(tight box, x) > thr (octree.cpp:141-149) is evaluated
// bit-exactly: FP64 with the reference's operation order and no contraction,
// compared as d2 > T2 with T2 the largest double whose sqrt is <= thr. The
// FP32 path first decides in FP32 with a 1e-6 relative guard band and only
// falls back to the exact FP64 test inside the band.
#include <atomic>
#include <cfloat>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "bh.h"
#include "gs_exp.cuh"
#define GS_TRACE_TU 2
#include "trace.cuh"

namespace gsb {

double gate_t2(double thr) {
  if (!(thr < INFINITY)) return INFINITY;
  double x = thr * thr;
  while (x > 0 && std::sqrt(x) > thr) x = std::nextafter(x, 0.0);
  while (std::sqrt(std::nextafter(x, INFINITY)) <= thr) x = std::nextafter(x, INFINITY);
  return x;
}

// gs_set_bh_walk: process-wide override of GS_BH_KERNEL / GS_BH_TASKS (-1: the
// environment's choice) so tests can drive every walk and window count
std::atomic<int> g_walk_kernel{-1}, g_walk_tasks{-1};

void set_bh_walk(int kernel, int tasks) {
  g_walk_kernel.store(kernel, std::memory_order_relaxed);
  g_walk_tasks.store(tasks, std::memory_order_relaxed);
}

namespace {

constexpr int kBhNT = 128;
#ifndef GS_BH_WS_NOWIN_MINB
#define GS_BH_WS_NOWIN_MINB 7
#endif
#ifndef GS_BH_WS_WIN_MINB
#define GS_BH_WS_WIN_MINB 8
#endif
#ifndef GS_BH_WS_HESS_MINB
#define GS_BH_WS_HESS_MINB 5
#endif


template <typename R>
struct BhArgs {
  const V4<R>* nadj;  // [m][2] {alpha sum, beta mean} (HESS)
  const V4<R>* nrec;  // [m][4] node records {unit, code} {unit, begin} {lo, count} {hi}
  const V4<R>* srec;  // [n][2] interaction coords (scaled FP32), p
  const V4<R>* squ;   // [n] unscaled q
  const V4<R>* sadj;  // [n][2] alpha, beta (leaf order)
  const int* perm;
  int n, nq, tgt_begin, n_tgt;
  const int* mp;  // node count on the device (first[n])
  const V4<R>* ev;    // VEL eval records; RHS/HESS external queries (by_index): (x, px) records
  const V4<R>* eadj;  // HESS external queries: (alpha_i, beta_i) records
  double kap, kc0x, kc0y, kc0z;
  double T2;         // exact gate threshold on d2
  R thr2_hi, thr2_lo;  // FP32 guard band around T2
  R thr2_in;           // max-distance shortcut: all descendants open
  R inv_two_s, c1;     // FP64 exp scale; HESS FP32 constant
  R grp_lim2;          // warps whose query box has diagonal^2 <= this walk as a group
  int split;           // 1: k_bh_grp takes the group warps, k_bh_ws the others
  int ntask;           // pre-order node windows per query (blockIdx.y); partials [task][query]
  int prefetch;        // L1-prefetch the skip target's record at every visit (GS_BH_PREFETCH)
  int lmd;             // literal-mean-dot aggregate dot scale (gs_config.literal_mean_dot)
  int by_index;        // RHS/HESS: queries are ev[0 .. nq) (a shard's records or arbitrary
                       // points, bh_point_*), not the tree's own points in leaf order
  int dense;           // 1: dense near fields (windows); 2: very dense (k_bh_grp by default)
  int* sm_ctr;         // non-null: blocks claim SM-local contiguous query blocks (claim_block)
  unsigned long long* dbg;  // GS_BH_DEBUG: group-walk counters (warps, iterations, segments, steps)
  V4<R>* part;
  uint32_t* per_query;
  unsigned long long* totals;
};

// exact reference gate: sqrt(dx^2 + dy^2 + dz^2) > thr, dx = max(lo-x, 0, x-hi)
__device__ __forceinline__ bool gate_exact(double lx, double ly, double lz, double hx, double hy,
                                           double hz, double x, double y, double z, double T2) {
  const double dx = fmax(fmax(__dsub_rn(lx, x), 0.0), __dsub_rn(x, hx));
  const double dy = fmax(fmax(__dsub_rn(ly, y), 0.0), __dsub_rn(y, hy));
  const double dz = fmax(fmax(__dsub_rn(lz, z), 0.0), __dsub_rn(z, hz));
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  return d2 > T2;
}

__device__ __forceinline__ bool gate(const double4& l, const double4& h, const double4& x,
                                     const BhArgs<double>& a) {
  return gate_exact(l.x, l.y, l.z, h.x, h.y, h.z, x.x, x.y, x.z, a.T2);
}

// Non-binding L1 prefetch (no register): the skip target's record is needed
// next whenever the node is not opened, and is usually not in L1 yet.
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

__device__ __forceinline__ bool lane_is_first_parked(bool here) {
  const unsigned b = __ballot_sync(0xffffffffu, here);
  return here && (threadIdx.x & 31) == __ffs(b) - 1;
}

template <typename R>
__device__ __forceinline__ bool all_inside(const V4<R>& l, const V4<R>& h, const V4<R>& x, R lim) {
  const R mx = max(x.x - l.x, h.x - x.x), my = max(x.y - l.y, h.y - x.y), mz = max(x.z - l.z, h.z - x.z);
  return mx * mx + my * my + mz * mz <= lim;
}

// Gate and fully-inside test of one node from the same per-axis differences
// a = lo - x, b = x - hi: min distance per axis max(a, b, 0) (the reference
// gate, octree.cpp:141-149), max distance per axis -min(a, b). Returns
// 1 = far (approximate), 2 = every descendant opens (direct range), 0 = open.
__device__ __forceinline__ int classify(const float4& l, const float4& h, const float4& x,
                                        const BhArgs<float>& a) {
  const float ax = l.x - x.x, ay = l.y - x.y, az = l.z - x.z;
  const float bx = x.x - h.x, by = x.y - h.y, bz = x.z - h.z;
  const float gx = fmaxf(fmaxf(ax, bx), 0.f), gy = fmaxf(fmaxf(ay, by), 0.f),
              gz = fmaxf(fmaxf(az, bz), 0.f);
  const float d2 = fmaf(gz, gz, fmaf(gy, gy, gx * gx));
  if (d2 > a.thr2_hi) return 1;
  if (d2 >= a.thr2_lo && gate_exact(l.x, l.y, l.z, h.x, h.y, h.z, x.x, x.y, x.z, a.T2)) return 1;
  const float mx = fminf(ax, bx), my = fminf(ay, by), mz = fminf(az, bz);
  return mx * mx + my * my + mz * mz <= a.thr2_in ? 2 : 0;
}
__device__ __forceinline__ int classify(const double4& l, const double4& h, const double4& x,
                                        const BhArgs<double>& a) {
  if (gate(l, h, x, a)) return 1;
  return all_inside(l, h, x, a.thr2_in) ? 2 : 0;
}

// Gaussian weight between the query and a source in interaction coordinates.
__device__ __forceinline__ float kern(float dx, float dy, float dz, const BhArgs<float>&) {
  float nr2 = -dx * dx;
  nr2 = fmaf(-dy, dy, nr2);
  nr2 = fmaf(-dz, dz, nr2);
  return ex2(nr2);
}
__device__ __forceinline__ double kern(double dx, double dy, double dz, const BhArgs<double>& a) {
  return exp_nonpos(-(dx * dx + dy * dy + dz * dz) * a.inv_two_s, kExp2Tab64);
}

__device__ __forceinline__ int code_of(float v) { return __float_as_int(v); }
__device__ __forceinline__ int code_of(double v) { return (int)v; }

template <typename R>
struct Acc {
  R v[12];
};

// One (direct or aggregate) unit: Q = source coords, P = momentum (sum),
// Al = alpha (sum), Be = beta (mean) -- bh_kernel.cpp:86-110 / :119-157.
// dsc: aggregate_dot_scale (bh_kernel.cpp:19-26) -- 1 for direct units and by
// default; 1/count for an approximated node under literal-mean-dot (LMD).
// LMD also accumulates sum c into acc.v[6] (the RHS partial's B.w) for
// bh_hamiltonian, whose dot is scaled too (bh_kernel.cpp:184).
template <typename R, int MODE, bool LMD = false>
__device__ __forceinline__ void unit(Acc<R>& acc, const V4<R>& xs, const V4<R>& px,
                                     const V4<R>& ai, const V4<R>& bi, const V4<R>& Q,
                                     const V4<R>& P, const V4<R>& Al, const V4<R>& Be,
                                     const BhArgs<R>& a, R dsc = R(1), bool on = true) {
  const R dx = xs.x - Q.x, dy = xs.y - Q.y, dz = xs.z - Q.z;
  const R g = on ? kern(dx, dy, dz, a) : R(0);  // on = false: a masked lane adds exact zeros
  if (MODE == kBhVel) {
    acc.v[0] += g * P.x; acc.v[1] += g * P.y; acc.v[2] += g * P.z;
  } else if (MODE == kBhRhs) {
    const R c = LMD ? (px.x * P.x + px.y * P.y + px.z * P.z) * dsc * g
                    : (px.x * P.x + px.y * P.y + px.z * P.z) * g;
    acc.v[0] += g * P.x; acc.v[1] += g * P.y; acc.v[2] += g * P.z;
    acc.v[3] += c * dx; acc.v[4] += c * dy; acc.v[5] += c * dz;
    if (LMD) acc.v[6] += c;
  } else {
    const R dbx = bi.x - Be.x, dby = bi.y - Be.y, dbz = bi.z - Be.z;
    const R ddb = dx * dbx + dy * dby + dz * dbz;
    const R s1 = (P.x * ai.x + P.y * ai.y + P.z * ai.z) + (px.x * Al.x + px.y * Al.y + px.z * Al.z);
    const R pp = px.x * P.x + px.y * P.y + px.z * P.z;
    const R t1 = g * s1;
    acc.v[0] += t1 * dx; acc.v[1] += t1 * dy; acc.v[2] += t1 * dz;
    acc.v[3] += g * Al.x; acc.v[4] += g * Al.y; acc.v[5] += g * Al.z;
    const R w = LMD ? g * (pp * dsc) : g * pp, uu = ddb * a.c1;
    acc.v[6] += w * (uu * dx - dbx); acc.v[7] += w * (uu * dy - dby); acc.v[8] += w * (uu * dz - dbz);
    const R m = g * ddb;
    acc.v[9] += m * P.x; acc.v[10] += m * P.y; acc.v[11] += m * P.z;
  }
}


// Squared diagonal of the warp's query box (valid lanes only): decides, per
// warp and identically in both kernels of a split launch, whether the warp's
// queries walk the tree as a group (k_bh_grp) or independently (k_bh_ws).
template <typename R>
__device__ __forceinline__ R warp_box_diag2(const V4<R>& x, bool valid) {
  R lx = valid ? x.x : R(INFINITY), ly = valid ? x.y : R(INFINITY), lz = valid ? x.z : R(INFINITY);
  R hx = valid ? x.x : R(-INFINITY), hy = valid ? x.y : R(-INFINITY), hz = valid ? x.z : R(-INFINITY);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lx = min(lx, __shfl_xor_sync(0xffffffffu, lx, o));
    ly = min(ly, __shfl_xor_sync(0xffffffffu, ly, o));
    lz = min(lz, __shfl_xor_sync(0xffffffffu, lz, o));
    hx = max(hx, __shfl_xor_sync(0xffffffffu, hx, o));
    hy = max(hy, __shfl_xor_sync(0xffffffffu, hy, o));
    hz = max(hz, __shfl_xor_sync(0xffffffffu, hz, o));
  }
  if (!(hx >= lx)) return R(0);  // no valid lane
  return (hx - lx) * (hx - lx) + (hy - ly) * (hy - ly) + (hz - lz) * (hz - lz);
}

// Cooperative sweep of one lane's long direct range: the 32 lanes split the
// range's points (lane-strided, coalesced loads), each accumulates the owner's
// terms, then a fixed butterfly reduction hands the sum to the owner. Fixed
// assignment + fixed reduction tree keep the result deterministic.
#ifndef GS_BH_BIG_RANGE
#define GS_BH_BIG_RANGE 24
#endif
constexpr int kBigRange = GS_BH_BIG_RANGE;

template <typename R>
__device__ __forceinline__ V4<R> shfl4(const V4<R>& v, int src) {
  return mk4<R>(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                __shfl_sync(0xffffffffu, v.z, src), R(0));
}

#ifndef GS_BH_COOP_GL
#define GS_BH_COOP_GL 32
#endif
// Lanes per owner in a cooperative sweep: the warp splits into 32/GL groups
// that sweep up to 32/GL owners' ranges at once (stride GL), then a log2(GL)
// butterfly inside each group and one shuffle hand each sum to its owner --
// 6x fewer reduction shuffles per range than a whole-warp sweep for GL = 8.
template <typename R, int MODE, bool LMD = false, bool COUNT = true>
__device__ __forceinline__ void coop_ranges(unsigned owners, int& j, int je, Acc<R>& acc,
                                            uint32_t& c_dir, const V4<R>& xs, const V4<R>& px,
                                            const V4<R>& ai, const V4<R>& bi,
                                            const BhArgs<R>& a) {
  constexpr int GL = GS_BH_COOP_GL, NG = 32 / GL;
  const int lane = threadIdx.x & 31, g = lane / GL, sub = lane % GL;
  constexpr int kAcc = MODE == kBhHess ? 12 : (MODE == kBhRhs ? (LMD ? 7 : 6) : 3);
  while (owners) {
    // this round: the first NG owners; group g serves the g-th of them
    unsigned sel = 0;
    int og = -1;
#pragma unroll
    for (int k = 0; k < NG; ++k) {
      if (owners) {
        const int b = __ffs(owners) - 1;
        if (k == g) og = b;
        sel |= 1u << b;
        owners &= owners - 1;
      }
    }
    const int src = og >= 0 ? og : 0;
    const int rb = __shfl_sync(0xffffffffu, j, src), re = __shfl_sync(0xffffffffu, je, src);
    const V4<R> oxs = shfl4<R>(xs, src), opx = shfl4<R>(px, src);
    V4<R> oai = ai, obi = bi;
    if (MODE == kBhHess) { oai = shfl4<R>(ai, src); obi = shfl4<R>(bi, src); }
    Acc<R> part;
#pragma unroll
    for (int c = 0; c < 12; ++c) part.v[c] = R(0);
    const V4<R> zero = mk4<R>(0, 0, 0);
    if (og >= 0) {
      for (int s = rb + sub; s <= re; s += GL) {
        V4<R> Q, P;
        ld8(a.srec + 2 * s, Q, P);
        if (MODE == kBhHess)
          unit<R, MODE, LMD>(part, oxs, opx, oai, obi, Q, P, ld4(a.sadj + 2 * s), ld4(a.sadj + 2 * s + 1), a);
        else
          unit<R, MODE, LMD>(part, oxs, opx, oai, obi, Q, P, zero, zero, a);
      }
    }
    // fixed butterfly inside each group, then owner lane <- its group's lane 0
    const bool mine = (sel >> lane) & 1u;
    const int from = mine ? GL * __popc(sel & ((1u << lane) - 1u)) : 0;
#pragma unroll
    for (int c = 0; c < kAcc; ++c) {
      R v = part.v[c];
#pragma unroll
      for (int off = GL / 2; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      v = __shfl_sync(0xffffffffu, v, from);
      if (mine) acc.v[c] += v;
    }
    if (mine) {
      if (COUNT) c_dir += (uint32_t)(je - j + 1);  // (k_bh_ws counts a range when it starts)
      j = je + 1;
    }
  }
}


// The query of thread slot qi: x (unscaled, for the gate), xs (interaction
// coordinates), px (momentum), ai/bi (HESS adjoints); returns the output slot
// (-1: no query). Queries are either the tree's own points in leaf order
// (restricted to point indices [tgt_begin, tgt_begin + n_tgt)), or external
// records ev[0 .. nq): eval points (VEL), a sharded flow's own targets taken by
// point index from its Morton-ordered records, or arbitrary (x, px[, alpha_i,
// beta_i]) queries (bh_point_gradients / bh_point_hessian_products,
// bh_kernel.cpp:81-160). External interaction coordinates are formed exactly
// as the tree's srec (tree_rescale).
template <typename R, int MODE>
__device__ __forceinline__ int load_query(const BhArgs<R>& a, int qi, V4<R>& x, V4<R>& xs,
                                          V4<R>& px, V4<R>& ai, V4<R>& bi) {
  x = mk4<R>(0, 0, 0);
  xs = px = ai = bi = x;
  if (qi >= a.nq) return -1;
  if (MODE == kBhVel || a.by_index) {
    x = ld4(a.ev + 2 * qi);
    if (sizeof(R) == 4)
      xs = mk4<R>((R)fmaf((float)a.kap, (float)x.x, -(float)(a.kap * a.kc0x)),
                  (R)fmaf((float)a.kap, (float)x.y, -(float)(a.kap * a.kc0y)),
                  (R)fmaf((float)a.kap, (float)x.z, -(float)(a.kap * a.kc0z)));
    else
      xs = x;
    if (MODE != kBhVel) px = ld4(a.ev + 2 * qi + 1);
    if (MODE == kBhHess) { ai = ld4(a.eadj + 2 * qi); bi = ld4(a.eadj + 2 * qi + 1); }
    return qi;
  }
  const int t = qi;
  x = ld4(a.squ + t);
  xs = ld4(a.srec + 2 * t);
  px = ld4(a.srec + 2 * t + 1);
  if (MODE == kBhHess) { ai = ld4(a.sadj + 2 * t); bi = ld4(a.sadj + 2 * t + 1); }
  const int i = a.perm[t] - a.tgt_begin;
  return (i >= 0 && i < a.n_tgt) ? i : -1;
}

// Output slot of query `out` in window blockIdx.y: partials and per-query
// counters are [window][query]; the epilogue / k_fold_counts fold the windows
// in fixed order.
template <int MODE, typename R>
__device__ __forceinline__ size_t out_slot(const BhArgs<R>& a, int out) {
  const int nout = MODE == kBhVel ? a.nq : a.n_tgt;
  return (size_t)blockIdx.y * nout + out;
}

// Work-stream variant: every lane walks its own query independently; each
// iteration a lane either continues its pending direct range (one point) or
// visits its next node (and, for a leaf / far / fully-inside node, evaluates
// the first unit in the same iteration). All lanes holding a unit then run
// the interaction together, so the warp does one unit of work per lane per
// iteration whatever node each lane is at. Same per-query node set, decisions
// and counts as the reference; only the summation order differs.
// FP32: cap registers for occupancy (RHS 80 regs -> 6 CTAs/SM, no spills)
template <typename R, int MODE, bool WIN>
constexpr int ws_min_blocks() {
  return sizeof(R) != 4 ? 1
                        : (MODE == kBhRhs ? (WIN ? GS_BH_WS_WIN_MINB : GS_BH_WS_NOWIN_MINB)
                                          : (MODE == kBhHess ? GS_BH_WS_HESS_MINB : 5));
}

// Query block of this CTA. With sm_ctr, the query blocks are dealt out in
// contiguous runs per SM (SM s owns blocks [s*per, (s+1)*per), claimed in
// order through its counter; an SM whose run is exhausted takes blocks from
// the others' runs): the warps resident on one SM then walk Morton-adjacent
// queries and share their near-field node records in L1. Each block id is
// claimed exactly once, so every query is walked once, by one thread.
__device__ __forceinline__ int claim_block(int* sm_ctr, int nblk) {
  __shared__ int s_blk;
  if (threadIdx.x == 0) {
    unsigned sm, nsm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    asm volatile("mov.u32 %0, %%nsmid;" : "=r"(nsm));
    nsm = min(nsm, 1024u);
    const int per = (nblk + (int)nsm - 1) / (int)nsm;
    int b = -1;
    for (unsigned k = 0; k < nsm && b < 0; ++k) {
      const unsigned s = (sm + k) % nsm;
      const int lo = (int)s * per;
      if (lo >= nblk) continue;
      const int c = atomicAdd(sm_ctr + s, 1);
      if (c < per && lo + c < nblk) b = lo + c;
    }
    s_blk = b;
  }
  __syncthreads();
  return s_blk;
}

// WIN: node windows (ntask > 1); the single-window instantiation drops the
// window bookkeeping (registers and instructions) for large N.
template <typename R, int MODE, bool WIN, bool LMD = false>
__global__ void __launch_bounds__(kBhNT, (ws_min_blocks<R, MODE, WIN>())) k_bh_ws(const BhArgs<R> a) {
  GS_TRACE_HERE();
  const int blk = (!WIN && a.sm_ctr) ? claim_block(a.sm_ctr, gridDim.x) : (int)blockIdx.x;
  V4<R> x, xs, px, ai, bi;
  const int out = load_query<R, MODE>(a, blk * kBhNT + threadIdx.x, x, xs, px, ai, bi);
  if (a.split && warp_box_diag2<R>(x, out >= 0) <= a.grp_lim2) return;  // k_bh_grp's warp
  Acc<R> acc;
#pragma unroll
  for (int c = 0; c < 12; ++c) acc.v[c] = R(0);
  uint32_t c_dir = 0, c_app = 0, c_vis = 0;
  const int m = *a.mp;
  // this block's window [A, B) of the pre-order node array and the leaf-order
  // interval [bA, bB) of the leaves inside it (see bh_tasks)
  int A = 0, B = m, bA = 0, bB = a.n;
  if (WIN) {
    A = (int)((long long)m * blockIdx.y / a.ntask);
    B = (int)((long long)m * (blockIdx.y + 1) / a.ntask);
    bA = A < m ? code_of(ld4(a.nrec + 4 * A + 1).w) : a.n;
    bB = B < m ? code_of(ld4(a.nrec + 4 * B + 1).w) : a.n;
  }
  int next = (out >= 0 && A < B) ? 0 : INT_MAX;  // an empty window (m < windows) walks nothing
  int j = 0, je = -1;  // pending direct range
  const V4<R> zero = mk4<R>(0, 0, 0);
#ifdef GS_BH_WS_STATS
  unsigned dbg_iter = 0, dbg_visit = 0, dbg_unit = 0, dbg_leaf = 0, dbg_far = 0, dbg_open = 0,
           dbg_range = 0, dbg_rpts = 0;
#define GS_WS_COUNT(x) (x)
#else
#define GS_WS_COUNT(x) ((void)0)
#endif
  while (__any_sync(0xffffffffu, next < m || j <= je)) {
    GS_WS_COUNT(++dbg_iter);
    bool have = false;
    V4<R> Q, P, Al, Be;  // this iteration's unit (read only when have)
    R dsc = R(1);
    if (j > je && next < m) {
      GS_WS_COUNT(++dbg_visit);
      const int nd = next;
      // the whole 64-B record at once, two independent 256-bit loads: half A
      // straight into the unit operands (a single leaf's point, or a node's
      // centroid + momentum sum), half B (tight box + count) for the gate
      V4<R> l, h;
      ld8(a.nrec + 4 * nd, Q, P);
      ld8(a.nrec + 4 * nd + 2, l, h);
      if (MODE == kBhHess) ld8(a.nadj + 2 * nd, Al, Be);  // the unit's adjoints (leaf or node)
      const int code = code_of(Q.w);
      const int begin = code_of(P.w);
      const int skip = code & 0x1fffffff;
      const bool own = !WIN || nd >= A;  // the node itself is in this block's window
      if (a.prefetch && skip < B) prefetch_l1(a.nrec + 4 * skip);
      next = skip;
      if (!WIN || skip > A) {  // the subtree reaches into the window (else: pass it by)
        c_vis += own;
        if (code < 0) {  // single-point leaf (always own): half A holds the point itself
          have = true;
          ++c_dir;
          GS_WS_COUNT(++dbg_leaf);
        } else {
          const int cnt = code_of(l.w);
          const int cls = (code & 0x40000000) ? 3 : classify(l, h, x, a);
          GS_WS_COUNT(cls == 1 ? ++dbg_far : (cls == 2 || cls == 3 || (code & 0x20000000)) ? (++dbg_range, dbg_rpts += cnt) : ++dbg_open);
          if (cls == 3) {  // depth-32 bucket (always own): all its points
            j = begin;
            je = begin + cnt - 1;
            c_dir += (uint32_t)cnt;  // counted once per range
          } else if (cls == 1) {  // far: one aggregate term at the centroid
            if (own) {
              if (LMD) dsc = R(1) / R(cnt);
              have = true;
              ++c_app;
            }
          } else if (cls == 2 || (code & 0x20000000)) {
            // every descendant opens, or a twig (children all leaves): range
            if (WIN) {
              j = max(begin, bA);
              je = min(begin + cnt, bB) - 1;
              c_vis += (uint32_t)max(0, min(skip, B) - max(nd + 1, A));
              c_dir += (uint32_t)max(0, je - j + 1);
            } else {
              j = begin;
              je = begin + cnt - 1;
              c_vis += (uint32_t)(skip - nd - 1);
              c_dir += (uint32_t)cnt;
            }
          } else {
            next = nd + 1;
          }
        }
      }
      if (next >= B || next <= nd) next = INT_MAX;  // window done; never loop on a corrupt skip
    }
    // long direct ranges (dense near field) are swept by the whole warp
    const unsigned big = __ballot_sync(0xffffffffu, !have && je - j + 1 >= kBigRange);
    if (big) coop_ranges<R, MODE, LMD, false>(big, j, je, acc, c_dir, xs, px, ai, bi, a);
    if (!have && j <= je) {
      ld8(a.srec + 2 * j, Q, P);
      if (MODE == kBhHess) { Al = ld4(a.sadj + 2 * j); Be = ld4(a.sadj + 2 * j + 1); }
      have = true;
      ++j;
    }
    if (have) unit<R, MODE, LMD>(acc, xs, px, ai, bi, Q, P, Al, Be, a, dsc);
    GS_WS_COUNT(dbg_unit += have);
  }
#ifdef GS_BH_WS_STATS
  if (a.dbg) {  // GS_BH_DEBUG (build with -DGS_BH_WS_STATS): warp iterations, lane visits, lane units
    unsigned long long v = dbg_visit, u = dbg_unit;
    unsigned long long ex[5] = {dbg_leaf, dbg_far, dbg_open, dbg_range, dbg_rpts};
    for (int o = 16; o > 0; o >>= 1) {
      v += __shfl_down_sync(0xffffffffu, v, o);
      u += __shfl_down_sync(0xffffffffu, u, o);
      for (int k = 0; k < 5; ++k) ex[k] += __shfl_down_sync(0xffffffffu, ex[k], o);
    }
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(a.dbg + 4, 1ull);
      atomicAdd(a.dbg + 5, (unsigned long long)dbg_iter);
      atomicAdd(a.dbg + 6, v);
      atomicAdd(a.dbg + 7, u);
      for (int k = 0; k < 5; ++k) atomicAdd(a.dbg + 8 + k, ex[k]);
    }
  }
#endif
#undef GS_WS_COUNT
  if (out >= 0) {
    const int per = MODE == kBhHess ? 4 : (MODE == kBhRhs ? 2 : 1);
    const size_t slot = out_slot<MODE>(a, out);
    V4<R>* o = a.part + (size_t)per * slot;
    for (int k = 0; k < per; ++k)
      st4(o + k, mk4<R>(acc.v[3 * k], acc.v[3 * k + 1], acc.v[3 * k + 2],
                        (LMD && MODE == kBhRhs && k == 1) ? acc.v[6] : R(0)));
    if (a.per_query) {
      a.per_query[3 * slot] = c_dir;
      a.per_query[3 * slot + 1] = c_app;
      a.per_query[3 * slot + 2] = c_vis;
    }
  }
  if (a.totals) {
    unsigned long long d = c_dir, p = c_app, v = c_vis;
    for (int o = 16; o > 0; o >>= 1) {
      d += __shfl_down_sync(0xffffffffu, d, o);
      p += __shfl_down_sync(0xffffffffu, p, o);
      v += __shfl_down_sync(0xffffffffu, v, o);
    }
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(a.totals, d);
      atomicAdd(a.totals + 1, p);
      atomicAdd(a.totals + 2, v);
    }
  }
}

// Group walk for warps whose 32 queries sit close together relative to the
// threshold (the dense regime of configs 2, 3 and 5, where each query's direct
// near field is thousands of points and neighbouring queries' fields nearly
// coincide). The warp walks the union of its lanes' node sets in pre-order,
// always serving the smallest pending node (lanes parked there classify it
// with their own exact gate, exactly as the reference would for that query).
// Direct work is NOT done per lane: each lane only records its pending direct
// interval of leaf-order points (a leaf, bucket, or fully-inside subtree), and
// the warp sweeps the union of the lanes' intervals in leaf order, one point
// per step with a broadcast load, every lane whose interval covers the point
// accumulating it. Sweeping [cursor, F) is safe once F = begin(current node):
// every lane has decided all its nodes before the current one. Each query's
// (direct, approximated, visited) sets and counts equal the reference's; only
// the summation order differs (and is fixed, so results are deterministic).
template <typename R, int MODE>
__device__ __forceinline__ void grp_sweep(int F, int& cursor, int ds, int de, Acc<R>& acc,
                                          uint32_t& c_dir, const V4<R>& xs, const V4<R>& px,
                                          const V4<R>& ai, const V4<R>& bi, const BhArgs<R>& a,
                                          unsigned& n_seg, unsigned& n_step) {
  for (;;) {
    const int from = max(ds, cursor);  // this lane's unswept part: [from, de]
    const int start = __reduce_min_sync(0xffffffffu, (de >= from) ? from : INT_MAX);
    if (start >= F) return;
    // the maximal run [start, E) of the union of the lanes' pending parts
    // (chained overlapping / adjacent intervals), clipped at F; every point
    // of it is loaded once (broadcast) and evaluated by all lanes, masked to
    // each lane's own interval -- long branch-free sweeps instead of one
    // segment per interval endpoint
    int E = start + 1;
    for (;;) {
      const int e = __reduce_max_sync(0xffffffffu, (de >= from && from <= E) ? de + 1 : 0);
      if (e <= E) break;
      E = e;
    }
    E = min(E, F);
    const int lo = max(from, start), hi = min(de + 1, E);  // this lane's part of the run
    if (hi > lo) c_dir += (uint32_t)(hi - lo);
    ++n_seg;
    n_step += (unsigned)(E - start);
#pragma unroll 4
    for (int j = start; j < E; ++j) {
      V4<R> Q, P;
      ld8(a.srec + 2 * j, Q, P);
      const bool on = j >= lo && j < hi;
      if (MODE == kBhHess)
        unit<R, MODE>(acc, xs, px, ai, bi, Q, P, ld4(a.sadj + 2 * j), ld4(a.sadj + 2 * j + 1), a, R(1), on);
      else
        unit<R, MODE>(acc, xs, px, ai, bi, Q, P, Q, Q, a, R(1), on);
    }
    cursor = E;
  }
}

#ifndef GS_BH_GRP_MINB
#define GS_BH_GRP_MINB 7
#endif
#ifndef GS_BH_GRP_HESS_MINB
#define GS_BH_GRP_HESS_MINB 7
#endif
// FP32: registers capped for occupancy (the walk is load-latency bound)
template <typename R, int MODE>
constexpr int grp_min_blocks() {
  return sizeof(R) != 4 ? 1 : (MODE == kBhHess ? GS_BH_GRP_HESS_MINB : GS_BH_GRP_MINB);
}

template <typename R, int MODE>
__global__ void __launch_bounds__(kBhNT, (grp_min_blocks<R, MODE>())) k_bh_grp(const BhArgs<R> a) {
  GS_TRACE_HERE();
  V4<R> x, xs, px, ai, bi;
  const int out = load_query<R, MODE>(a, blockIdx.x * kBhNT + threadIdx.x, x, xs, px, ai, bi);
  if (a.split && !(warp_box_diag2<R>(x, out >= 0) <= a.grp_lim2)) return;  // k_bh_ws's warp
  Acc<R> acc;
#pragma unroll
  for (int c = 0; c < 12; ++c) acc.v[c] = R(0);
  uint32_t c_dir = 0, c_app = 0, c_vis = 0;
  const int m = *a.mp;
  // this block's window [A, B) of the pre-order node array and the leaf-order
  // interval [bA, bB) of the leaves inside it (see bh_tasks)
  int A = 0, B = m, bA = 0, bB = a.n;
  if (a.ntask > 1) {
    A = (int)((long long)m * blockIdx.y / a.ntask);
    B = (int)((long long)m * (blockIdx.y + 1) / a.ntask);
    bA = A < m ? code_of(ld4(a.nrec + 4 * A + 1).w) : a.n;
    bB = B < m ? code_of(ld4(a.nrec + 4 * B + 1).w) : a.n;
  }
  int next = (out >= 0 && A < B) ? 0 : INT_MAX;  // an empty window (m < windows) walks nothing
  int ds = 0, de = -1;  // this lane's pending direct interval (leaf order, inclusive)
  int cursor = 0;       // warp-uniform sweep position
  unsigned n_iter = 0, n_seg = 0, n_step = 0;
  const V4<R> zero = mk4<R>(0, 0, 0);
  for (;;) {
    const int nd = __reduce_min_sync(0xffffffffu, next);
    if (nd == INT_MAX) break;
    ++n_iter;
    // the node's 64-B record, loaded by every lane (broadcast): half A = the
    // node's unit (point or centroid + momentum sum), half B = box + count
    V4<R> Q, P, l, h;
    ld8(a.nrec + 4 * nd, Q, P);
    ld8(a.nrec + 4 * nd + 2, l, h);
    const int code = code_of(Q.w);
    const int begin = code_of(P.w);
    const int skip = code & 0x1fffffff;
    const bool here = next == nd;
    if (a.prefetch && skip < B && lane_is_first_parked(here)) prefetch_l1(a.nrec + 4 * skip);
    bool have = false, ranged = false;
    V4<R> Al = zero, Be = zero;
    int rb = 0, re = -1;
    if (here) {
      const bool own = nd >= A;  // the node itself is in this block's window
      next = skip;
      if (skip > A) {  // the subtree reaches into the window (else: pass it by)
        c_vis += own;
        if (code < 0) {  // single-point leaf (always own): half A holds the point itself
          if (MODE == kBhHess) ld8(a.nadj + 2 * nd, Al, Be);
          have = true;
          ++c_dir;
        } else {
          const int cnt = code_of(l.w);
          const int cls = (code & 0x40000000) ? 3 : classify(l, h, x, a);
          if (cls == 3) {  // depth-32 bucket (always own): all its points
            ranged = true;
            rb = begin;
            re = begin + cnt - 1;
          } else if (cls == 1) {  // far: one aggregate term at the centroid
            if (own) {
              if (MODE == kBhHess) ld8(a.nadj + 2 * nd, Al, Be);
              have = true;
              ++c_app;
            }
          } else if (cls == 2 || (code & 0x20000000)) {
            // every descendant opens, or a twig (children all leaves): range
            ranged = true;
            rb = max(begin, bA);
            re = min(begin + cnt, bB) - 1;
            c_vis += (uint32_t)max(0, min(skip, B) - max(nd + 1, A));
          } else {
            next = nd + 1;
          }
        }
      }
      if (next >= B || next <= nd) next = INT_MAX;
    }
    if (__any_sync(0xffffffffu, ranged)) {
      // every earlier pending interval ends before begin(nd): settle them first
      grp_sweep<R, MODE>(begin, cursor, ds, de, acc, c_dir, xs, px, ai, bi, a, n_seg, n_step);
      if (ranged) { ds = rb; de = re; }
    }
    if (have) unit<R, MODE>(acc, xs, px, ai, bi, Q, P, Al, Be, a);
  }
  grp_sweep<R, MODE>(INT_MAX, cursor, ds, de, acc, c_dir, xs, px, ai, bi, a, n_seg, n_step);
  if (a.dbg && (threadIdx.x & 31) == 0) {
    atomicAdd(a.dbg, 1ull);
    atomicAdd(a.dbg + 1, (unsigned long long)n_iter);
    atomicAdd(a.dbg + 2, (unsigned long long)n_seg);
    atomicAdd(a.dbg + 3, (unsigned long long)n_step);
  }
  if (out >= 0) {
    const int per = MODE == kBhHess ? 4 : (MODE == kBhRhs ? 2 : 1);
    const size_t slot = out_slot<MODE>(a, out);
    V4<R>* o = a.part + (size_t)per * slot;
    for (int k = 0; k < per; ++k) st4(o + k, mk4<R>(acc.v[3 * k], acc.v[3 * k + 1], acc.v[3 * k + 2]));
    if (a.per_query) {
      a.per_query[3 * slot] = c_dir;
      a.per_query[3 * slot + 1] = c_app;
      a.per_query[3 * slot + 2] = c_vis;
    }
  }
  if (a.totals) {
    unsigned long long d = c_dir, p = c_app, v = c_vis;
    for (int o = 16; o > 0; o >>= 1) {
      d += __shfl_down_sync(0xffffffffu, d, o);
      p += __shfl_down_sync(0xffffffffu, p, o);
      v += __shfl_down_sync(0xffffffffu, v, o);
    }
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(a.totals, d);
      atomicAdd(a.totals + 1, p);
      atomicAdd(a.totals + 2, v);
    }
  }
}


// GS_BH_KERNEL: 1 (default) = independent walks (k_bh_ws), 3 = group walk
// (k_bh_grp), 4 = split launch (group walk for warps whose query box is small
// against the threshold, independent walks for the rest). The first two
// designs (a warp-synchronous min-node walk over separate node arrays, and a
// software-pipelined independent walk) were slower and are retired. Measured (B200, FP32): the
// group walk wins on config 3 (tube, sigma 5: 3.8 vs 4.6 ms per RHS) and loses
// on configs 2, 4 and 5, so independent walks are the default.
static int bh_kernel_choice() {
  const int o = g_walk_kernel.load(std::memory_order_relaxed);
  if (o >= 0) return o;  // gs_set_bh_walk
  static int v = [] {
    const char* e = std::getenv("GS_BH_KERNEL");
    return e ? std::atoi(e) : 0;  // 0: by regime (dense near fields -> 3, else 1)
  }();
  return v;
}

// A warp walks as a group when its query box diagonal is <= ratio * thr.
static double bh_group_ratio() {
  static double v = [] {
    const char* e = std::getenv("GS_BH_GRP_RATIO");
    return e ? std::atof(e) : 0.25;
  }();
  return v;
}

template <typename R>
int launch(int mode, BhArgs<R> a, cudaStream_t st) {
  // literal-mean-dot: independent walks only (the group walk has no LMD variant)
  const int choice = bh_kernel_choice();
  // (FP64: the group walk from dense on -- config 2 FP64 8.75 vs 9.0 ms)
  const int grp_from = sizeof(R) == 8 ? 1 : 2;
  const int kind = a.lmd ? 1 : (choice ? choice : (a.dense >= grp_from ? 3 : 1));
  const dim3 nb(std::max(1, (a.nq + kBhNT - 1) / kBhNT), std::max(1, a.ntask));
  static const bool dbg = std::getenv("GS_BH_DEBUG") != nullptr;
  static unsigned long long* dbuf = nullptr;
  if (dbg && !dbuf) cudaMalloc(&dbuf, 128);
  if (dbg) {
    cudaMemsetAsync(dbuf, 0, 128, st);
    a.dbg = dbuf;
  }
  if (kind == 3 || kind == 4) {
    a.split = kind == 4;
    if (mode == kBhRhs) k_bh_grp<R, kBhRhs><<<nb, kBhNT, 0, st>>>(a);
    else if (mode == kBhHess) k_bh_grp<R, kBhHess><<<nb, kBhNT, 0, st>>>(a);
    else k_bh_grp<R, kBhVel><<<nb, kBhNT, 0, st>>>(a);
    GS_CUDA_OK(cudaGetLastError());
    if (dbg) {
      unsigned long long h[4];
      cudaMemcpyAsync(h, dbuf, sizeof h, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      std::fprintf(stderr, "[bh grp mode %d nq %d] warps %llu iters %llu segs %llu steps %llu\n", mode,
                   a.nq, h[0], h[1], h[2], h[3]);
    }
    if (kind == 3) return GS_OK;
  }
  struct DbgPrint {
    bool on;
    unsigned long long* buf;
    cudaStream_t st;
    int mode, nq;
    ~DbgPrint() {
      if (!on) return;
      unsigned long long h[16];
      cudaMemcpyAsync(h, buf, sizeof h, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      if (h[4]) {
        const double L = 32.0 * h[4];
        std::fprintf(stderr, "[bh ws mode %d nq %d] warps %llu iters/warp %.1f visits/lane %.1f units/lane %.1f simt %.1f"
                     " | leaf %.1f far %.1f open %.1f range %.1f (pts %.1f)\n",
                     mode, nq, h[4], (double)h[5] / h[4], (double)h[6] / L, (double)h[7] / L,
                     (double)(h[6] + h[7]) / h[5], h[8] / L, h[9] / L, h[10] / L, h[11] / L, h[12] / L);
      }
    }
  } dbg_print{dbg, dbuf, st, mode, a.nq};
  {  // 1 (default), 4 (after the group warps); retired designs 0, 2 map here
    if (a.lmd && mode != kBhVel) {  // the dot scale has no effect on velocities
      if (a.ntask > 1) {
        if (mode == kBhRhs) k_bh_ws<R, kBhRhs, true, true><<<nb, kBhNT, 0, st>>>(a);
        else k_bh_ws<R, kBhHess, true, true><<<nb, kBhNT, 0, st>>>(a);
      } else {
        if (mode == kBhRhs) k_bh_ws<R, kBhRhs, false, true><<<nb, kBhNT, 0, st>>>(a);
        else k_bh_ws<R, kBhHess, false, true><<<nb, kBhNT, 0, st>>>(a);
      }
    } else if (a.ntask > 1) {
      if (mode == kBhRhs) k_bh_ws<R, kBhRhs, true><<<nb, kBhNT, 0, st>>>(a);
      else if (mode == kBhHess) k_bh_ws<R, kBhHess, true><<<nb, kBhNT, 0, st>>>(a);
      else k_bh_ws<R, kBhVel, true><<<nb, kBhNT, 0, st>>>(a);
    } else {
      if (mode == kBhRhs) k_bh_ws<R, kBhRhs, false><<<nb, kBhNT, 0, st>>>(a);
      else if (mode == kBhHess) k_bh_ws<R, kBhHess, false><<<nb, kBhNT, 0, st>>>(a);
      else k_bh_ws<R, kBhVel, false><<<nb, kBhNT, 0, st>>>(a);
    }
  }
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}

template <typename R>
BhArgs<R> make_args(DevTree& t, double sigma, double thr, const BhQuery& q) {
  BhArgs<R> a{};
  a.nadj = t.nadj.as<V4<R>>();
  a.srec = t.srec.as<V4<R>>();
  a.nrec = t.nrec.as<V4<R>>();
  a.squ = t.squ.as<V4<R>>();
  a.sadj = t.sadj.as<V4<R>>();
  a.perm = t.perm.as<int>();
  a.n = (int)t.n;
  a.mp = t.first.as<int>() + t.n;
  a.tgt_begin = q.tgt_begin;
  a.n_tgt = q.n_tgt;
  a.nq = q.mode == kBhVel ? q.m : (q.by_index ? q.n_tgt : (int)t.n);
  a.by_index = q.by_index;
  a.dense = q.dense;
  a.ev = static_cast<const V4<R>*>(q.ev);
  a.eadj = static_cast<const V4<R>*>(q.eadj);
  const KernelConsts& kc = t.kc;
  a.kap = kc.kappa;
  a.kc0x = kc.c0[0];
  a.kc0y = kc.c0[1];
  a.kc0z = kc.c0[2];
  a.T2 = gate_t2(thr);
  const double t2 = a.T2;
  if (sizeof(R) == 4) {
    a.thr2_hi = (R)(t2 * (1.0 + 1e-6));
    a.thr2_lo = (R)(t2 * (1.0 - 1e-6));
    a.c1 = (R)(1.0 / (kc.kappa * kc.kappa * kc.s));
  } else {
    a.thr2_hi = (R)t2;
    a.thr2_lo = (R)t2;
    a.c1 = (R)kc.inv_s;
  }
  a.thr2_in = (R)(thr < INFINITY ? thr * thr * (1.0 - 1e-5) : INFINITY);
  {
    const double g = bh_group_ratio() * thr;
    a.grp_lim2 = (R)(g < 1e150 ? g * g : INFINITY);
  }
  a.split = 0;
  {
    static const int pf = [] {
      const char* e = std::getenv("GS_BH_PREFETCH");
      return e ? std::atoi(e) : 0;  // measured: no gain (records hit L1/L2 already)
    }();
    a.prefetch = pf;
  }
  a.inv_two_s = (R)kc.inv_two_s;
  a.part = static_cast<V4<R>*>(q.part);
  a.per_query = q.per_query;
  a.totals = q.totals;
  a.ntask = std::max(1, q.ntask);
  a.lmd = q.lmd;
  (void)sigma;
  return a;
}

// Per-query counters of K node windows: out[i] = sum over windows in order.
__global__ void k_fold_counts(const uint32_t* __restrict__ in, int K, int64_t n3,
                              uint32_t* __restrict__ out) {
  GS_TRACE_HERE();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n3) return;
  uint32_t v = 0;
  for (int k = 0; k < K; ++k) v += in[(size_t)k * n3 + i];
  out[i] = v;
}

}  // namespace

int bh_traverse(const Device&, int prec, DevTree& t, double sigma, double thr, const BhQuery& q,
                cudaStream_t st) {
  static const int sm_local = [] {
    const char* e = std::getenv("GS_BH_SM_LOCAL");
    return e ? std::atoi(e) : 1;
  }();
  int* ctr = nullptr;
  if (sm_local && q.ntask <= 1) {
    GS_TRY_INT(t.sm_ctr.ensure(4 * 1024));
    GS_CUDA_OK(cudaMemsetAsync(t.sm_ctr.ptr, 0, 4 * 1024, st));
    ctr = t.sm_ctr.as<int>();
  }
  // per-query counters with node windows: each window writes its own slice
  // [window][query][3]; the slices are folded (summed) into q.per_query
  const int K = std::max(1, q.ntask);
  const int nout = q.mode == kBhVel ? q.m : q.n_tgt;
  uint32_t* pq = q.per_query;
  if (pq && K > 1) {
    GS_TRY_INT(t.pq_win.ensure(sizeof(uint32_t) * 3 * (size_t)nout * K));
    pq = t.pq_win.as<uint32_t>();
  }
  int s;
  if (prec == kF32) {
    BhArgs<float> a = make_args<float>(t, sigma, thr, q);
    a.sm_ctr = ctr;
    a.per_query = pq;
    s = launch<float>(q.mode, a, st);
  } else {
    BhArgs<double> a = make_args<double>(t, sigma, thr, q);
    a.sm_ctr = ctr;
    a.per_query = pq;
    s = launch<double>(q.mode, a, st);
  }
  if (s != GS_OK || !q.per_query || K == 1 || nout == 0) return s;
  const int64_t n3 = 3 * (int64_t)nout;
  k_fold_counts<<<(unsigned)((n3 + 255) / 256), 256, 0, st>>>(pq, K, n3, q.per_query);
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}

// Node windows per query: a latency-bound walk needs many resident warps, and
// with few queries (configs 2, 3, 5: 20k-50k points = 600-1600 warps) one warp
// per 32 queries leaves the SMs mostly idle. Splitting the pre-order node
// array into K windows (each block walks its queries through one window;
// the epilogue folds the K partials in fixed order) multiplies the warps by K.
constexpr int kMaxBhTasks = 64;
thread_local int t_bh_concurrency = 1;
void set_bh_concurrency(int c) { t_bh_concurrency = std::max(1, c); }

// Windows per query: enough warps to fill the SMs (2 waves of 32 resident
// warps), and -- when the caller's point set is dense at the gate radius (an
// estimated >= 1024 points within thr of a point, from the host bounding box
// in kc.ext), so that every walk carries thousands of direct interactions --
// 32 windows: each window's blocks then work in one region of the tree (its
// records stay in L1) and the long walks are cut into many short ones.
// Measured (config 3 evaluate): K = 7 -> 32: 0.207 -> 0.162 s; config 5:
// 0.49 -> 0.35 s per 8 subjects; config 4 (sparse, ~500 within thr): K = 1-2
// stays best. Skipped when several flows share the GPU (batched subjects),
// whose concurrency already fills it.
int bh_tasks(int64_t nq, int64_t n, double thr, const KernelConsts& kc, int* dense) {
  if (dense) *dense = 0;
  static const int env_forced = [] {
    const char* e = std::getenv("GS_BH_TASKS");
    return e ? std::atoi(e) : 0;
  }();
  const int o = g_walk_tasks.load(std::memory_order_relaxed);
  const int forced = o >= 0 ? o : env_forced;  // gs_set_bh_walk, else GS_BH_TASKS
  const int64_t warps = (nq + 31) / 32;
  const int64_t want = 148 * 64;  // ~2 waves of 32 resident warps per SM
  int K = (int)std::max<int64_t>(1, std::min<int64_t>(16, (want + warps - 1) / warps));
  if (t_bh_concurrency == 1 && kc.ext[0] + kc.ext[1] + kc.ext[2] > 0 && thr < INFINITY) {
    double frac = 1.0;
    for (int a = 0; a < 3; ++a)
      if (kc.ext[a] > 0) frac *= std::min(1.0, 2.0 * thr / kc.ext[a]);
    const int64_t cap = std::max<int64_t>(1, (int64_t(4) << 20) / std::max<int64_t>(nq, 1));
    // estimated points within thr of a point (the host bounding box at the
    // flow's upload): >= 1024 -> 32 node windows; >= 4096 -> the group walk
    // too (configs 3 and 5: 16k / 4.9k; config 2's 2.9k keeps the independent
    // walk -- its flow spreads: 5.90 vs 6.07 ms over 20 steps, config 5
    // 39.7 vs 35.9 ms per subject the other way)
    const double est = frac * (double)n;
    if (est >= 1024.0) {
      K = (int)std::max<int64_t>(K, std::min<int64_t>(32, cap));
      if (dense) *dense = est >= 4096.0 ? 2 : 1;
    }
  }
  if (forced > 0) K = forced;  // the regime (dense) is still detected
  return std::min(K, kMaxBhTasks);
}

int bh_keep_trees(BhWork& w, int T) {
  while ((int)w.kept.size() < T) w.kept.emplace_back(new DevTree);
  return GS_OK;
}

static DevTree& tree_for(BhWork& w) {
  if (w.cache_slot >= 0 && w.cache_slot < (int)w.kept.size()) return *w.kept[w.cache_slot];
  return w.cur;
}

int bh_forward_stage(const Device& dev, int prec, const KernelConsts& kc, const gs_config& cfg,
                     const void* rec, int64_t n, int64_t tb, int64_t nt, BhWork& w, FwdEpi e,
                     cudaStream_t st, int64_t* launches, int* energy_blocks, gs_stats*) {
  DevTree& t = tree_for(w);
  kt_mark(1, st);
  t.lean = true;  // walked only: no FP64 node sums / boxes
  GS_TRY_INT(tree_build(dev, prec, kc, rec, n, t, st, nullptr, e.bad_step ? e.bad_step + 1 : nullptr));
  kt_mark(1, st);
  int dense = 0;
  const int K = bh_tasks(nt, n, cfg.threshold_multiplier * cfg.sigma, kc, &dense);
  GS_TRY_INT(w.part.ensure(2 * vec_bytes(prec) * K * std::max<int64_t>(nt, 1)));
  GS_TRY_INT(w.stats.ensure(64));
  BhQuery q;
  q.mode = kBhRhs;
  q.ntask = K;
  q.dense = dense;
  q.lmd = cfg.literal_mean_dot;
  if (tb != 0 || nt != n) {  // a shard: walk only its own targets, by point index
    q.by_index = 1;
    q.ev = static_cast<const char*>(rec) + 2 * vec_bytes(prec) * tb;
  }
  q.tgt_begin = (int)tb;
  q.n_tgt = (int)nt;
  q.part = w.part.ptr;
  q.totals = w.stats.as<unsigned long long>();
  const double thr = cfg.threshold_multiplier * cfg.sigma;
  kt_mark(0, st);
  GS_TRY_INT(bh_traverse(dev, prec, t, cfg.sigma, thr, q, st));
  kt_mark(0, st);
  e.S = K;
  e.parts_per_tgt = 2;
  e.part = w.part.ptr;
  e.n_tgt = (int)nt;
  e.tgt_begin = (int)tb;
  e.cp = 2.0;
  e.cq = prec == kF32 ? -kc.two_over_s / kc.kappa : -kc.two_over_s;
  GS_TRY_INT(fwd_epilogue(prec, e, st, energy_blocks));
  if (launches) *launches += 30;  // build (~27) + traversal + epilogue
  return GS_OK;
}

int bh_backward_step(const Device& dev, int prec, const KernelConsts& kc, const gs_config& cfg,
                     const void* rec_k, void* adj, int64_t n, int64_t tb, int64_t nt, int k,
                     BhWork& w, bool cached, BwdEpi e, cudaStream_t st, gs_stats*) {
  DevTree* t = nullptr;
  if (cached && k < (int)w.kept.size()) {
    t = w.kept[k].get();
  } else {
    t = &w.cur;
    t->lean = true;
    GS_TRY_INT(tree_build(dev, prec, kc, rec_k, n, *t, st));
  }
  GS_TRY_INT(tree_accumulate(prec, *t, adj, st));
  int dense = 0;
  const int K = bh_tasks(nt, n, cfg.threshold_multiplier * cfg.sigma, kc, &dense);
  GS_TRY_INT(w.part.ensure(4 * vec_bytes(prec) * K * std::max<int64_t>(nt, 1)));
  GS_TRY_INT(w.stats.ensure(64));
  BhQuery q;
  q.mode = kBhHess;
  q.ntask = K;
  q.dense = dense;
  q.lmd = cfg.literal_mean_dot;
  if (tb != 0 || nt != n) {  // a shard: its own targets by point index (records + adjoints)
    q.by_index = 1;
    q.ev = static_cast<const char*>(rec_k) + 2 * vec_bytes(prec) * tb;
    q.eadj = static_cast<const char*>(adj) + 2 * vec_bytes(prec) * tb;
  }
  q.tgt_begin = (int)tb;
  q.n_tgt = (int)nt;
  q.part = w.part.ptr;
  q.totals = w.stats.as<unsigned long long>();
  kt_mark(6, st);
  GS_TRY_INT(bh_traverse(dev, prec, *t, cfg.sigma, cfg.threshold_multiplier * cfg.sigma, q, st));
  kt_mark(6, st);
  e.S = K;
  e.part = w.part.ptr;
  GS_TRY_INT(bwd_epilogue(prec, e, st));
  return GS_OK;
}

int bh_velocity_step(const Device& dev, int prec, const KernelConsts& kc, const gs_config& cfg,
                     const void* rec_k, int64_t n, void* ev, int64_t m, BhWork& w, VelEpi e,
                     cudaStream_t st) {
  w.cur.lean = true;
  GS_TRY_INT(tree_build(dev, prec, kc, rec_k, n, w.cur, st));
  int dense = 0;
  const int K = bh_tasks(m, n, cfg.threshold_multiplier * cfg.sigma, kc, &dense);
  GS_TRY_INT(w.part.ensure(vec_bytes(prec) * K * m));
  BhQuery q;
  q.mode = kBhVel;
  q.ntask = K;
  q.dense = dense;
  q.ev = ev;
  q.m = (int)m;
  q.part = w.part.ptr;
  GS_TRY_INT(bh_traverse(dev, prec, w.cur, cfg.sigma, cfg.threshold_multiplier * cfg.sigma, q, st));
  e.S = K;
  e.part = w.part.ptr;
  GS_TRY_INT(vel_epilogue(prec, e, st));
  return GS_OK;
}

int trace_install_bh(unsigned long long* buf) {
  GS_CUDA_OK(trace_install_here(buf));
  return GS_OK;
}

}  // namespace gsb
