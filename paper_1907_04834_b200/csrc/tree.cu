// tree.cu -- octree build on sm_100a: bbox -> midpoint-replay Morton keys ->
// LSD radix sort -> radix-tree topology collapsed to the reference octree ->
// bottom-up aggregates.
//
// The reference builds its octree by sequential pointer insertion
// (octree.cpp:74-117). Its node set is fully determined by the points:
//   * the root cell is the bounding box padded by 1e-9 * extent (octree.cpp:9,25-40);
//   * a child cell is an octant of its parent's cell split at the FP64
//     midpoint c = 0.5 * (lo + hi), points on the plane going high
//     (octant_of :42-45, make_child :59-72);
//   * a cell exists iff it is the root, or its parent holds >= 2 points and it
//     holds >= 1; it is a leaf iff it holds 1 point or sits at depth 32
//     (bucket, :93-97).
// So with key = the 3-bit octant digits of every level (replayed per axis in
// FP64 exactly as the reference computes them), the cells are the distinct
// key prefixes shared by >= 2 points plus one leaf per point (or bucket), and
// a depth-first walk of the reference tree with children 0..7 visits the
// points in sorted-key order. With L[t] = common digits of sorted keys t and
// t+1, position a starts the internal nodes of levels L[a-1]+1 .. min(L[a],31)
// and one leaf; ordering nodes by (start, level) is the depth-first pre-order.
// Everything below is that construction, one thread per position/node.
#include <chrono>
#include <cstdlib>

#include <cooperative_groups.h>
#include <cuda/atomic>

#include "bh.h"
#define GS_TRACE_TU 1
#include "trace.cuh"

namespace gsb {

namespace {

constexpr int kNT = 256;

inline int nblocks(int64_t n, int nt) { return (int)std::max<int64_t>(1, (n + nt - 1) / nt); }

// ------------------------------------------------------------------ bbox ---
// root = [lo - pad, hi + pad], pad = 1e-9 * (hi - lo)   (octree.cpp:9,27-35)
__device__ void bbox_root(const double* part, int nb, double* root) {
  __shared__ double s[6][kNT / 32];
  double v[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
  for (int b = threadIdx.x; b < nb; b += kNT)
#pragma unroll
    for (int a = 0; a < 6; ++a) v[a] = a < 3 ? fmin(v[a], part[6 * b + a]) : fmax(v[a], part[6 * b + a]);
#pragma unroll
  for (int a = 0; a < 6; ++a) {
    for (int o = 16; o > 0; o >>= 1) {
      const double w = __shfl_down_sync(0xffffffffu, v[a], o);
      v[a] = a < 3 ? fmin(v[a], w) : fmax(v[a], w);
    }
    if ((threadIdx.x & 31) == 0) s[a][threadIdx.x >> 5] = v[a];
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    const int a = threadIdx.x;
    double lo = s[a][0], hi = s[3 + a][0];
    for (int w = 1; w < kNT / 32; ++w) {
      lo = fmin(lo, s[a][w]);
      hi = fmax(hi, s[3 + a][w]);
    }
    const double pad = __dmul_rn(__dsub_rn(hi, lo), 1e-9);
    root[a] = __dsub_rn(lo, pad);
    root[3 + a] = __dadd_rn(hi, pad);
  }
}

template <typename R>
__global__ void __launch_bounds__(kNT) k_bbox(const V4<R>* rec, int64_t n, double* part,
                                              unsigned* done, double* root) {
  GS_PDL_ENTRY();
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
    const V4<R> q = ld4(rec + 2 * i);
    const double v[3] = {(double)q.x, (double)q.y, (double)q.z};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = fmin(lo[a], v[a]);
      hi[a] = fmax(hi[a], v[a]);
    }
  }
  __shared__ double s[6][kNT / 32];
  __shared__ bool s_last;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fmin(lo[a], __shfl_down_sync(0xffffffffu, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_down_sync(0xffffffffu, hi[a], o));
    }
    if ((threadIdx.x & 31) == 0) {
      s[a][threadIdx.x >> 5] = lo[a];
      s[3 + a][threadIdx.x >> 5] = hi[a];
    }
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double r = s[threadIdx.x][0];
    for (int w = 1; w < kNT / 32; ++w)
      r = threadIdx.x < 3 ? fmin(r, s[threadIdx.x][w]) : fmax(r, s[threadIdx.x][w]);
    part[6 * blockIdx.x + threadIdx.x] = r;
  }
  // the last block to finish reduces the partials to the padded root box (the
  // arrival counter resets itself for the next build)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) *done = 0;
  bbox_root(part, gridDim.x, root);
}


// ------------------------------------------------------------------ keys ---
// Levels 1..21 -> key_hi (63 bits, level 1 most significant), 22..32 -> key_lo
// (33 bits). key_lo only orders points that share all 21 levels of key_hi: the
// sort uses it for those runs only. Where the previous build had such runs (a
// diverged flow puts most points in them) computing it here (11 more levels
// of the same replay, +12 us at 1M) is cheaper than replaying 32 levels per
// run member later; otherwise the tie sort replays it for its few members.
template <typename R>
__global__ void __launch_bounds__(kNT) k_keys(const V4<R>* rec, int64_t n, const double* root,
                                              uint64_t* kh, uint64_t* kl, const unsigned* want_lo,
                                              unsigned* lo_valid) {
  GS_PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
  if (i >= n) return;
  const V4<R> q = ld4(rec + 2 * i);
  const double x[3] = {(double)q.x, (double)q.y, (double)q.z};
  double lo[3] = {root[0], root[1], root[2]}, hi[3] = {root[3], root[4], root[5]};
  uint64_t h = 0;
#pragma unroll
  for (int lev = 1; lev <= 21; ++lev) {
    unsigned dig = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double c = __dmul_rn(0.5, __dadd_rn(lo[a], hi[a]));
      const bool up = x[a] >= c;
      lo[a] = up ? c : lo[a];
      hi[a] = up ? hi[a] : c;
      dig |= (unsigned)up << a;
    }
    h = (h << 3) | dig;
  }
  kh[i] = h;
  // the deep key when the previous build of this tree had ties (want_lo: its
  // tie flag, still in the sort scratch; null: unknown -> yes); else the tie
  // sort replays it for run members itself (k_tie_sort, lo_valid = 0)
  const bool do_lo = want_lo == nullptr || *want_lo != 0;
  if (i == 0) *lo_valid = do_lo ? 1u : 0u;
  if (!do_lo) return;
  uint64_t l = 0;
#pragma unroll
  for (int lev = 22; lev <= 32; ++lev) {
    unsigned dig = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double c = __dmul_rn(0.5, __dadd_rn(lo[a], hi[a]));
      const bool up = x[a] >= c;
      lo[a] = up ? c : lo[a];
      hi[a] = up ? hi[a] : c;
      dig |= (unsigned)up << a;
    }
    l = (l << 3) | dig;
  }
  kl[i] = l;
}

// levels 22..32 of point x whose levels 1..21 are h: the level-21 cell is
// replayed from h's digits (the same midpoints as the comparisons produced)
__device__ __forceinline__ uint64_t key_lo_of(const double x[3], uint64_t h, const double* root) {
  double lo[3] = {root[0], root[1], root[2]}, hi[3] = {root[3], root[4], root[5]};
  for (int lev = 1; lev <= 21; ++lev) {
    const unsigned dig = (unsigned)(h >> (3 * (21 - lev))) & 7u;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double c = __dmul_rn(0.5, __dadd_rn(lo[a], hi[a]));
      if ((dig >> a) & 1u) lo[a] = c;
      else hi[a] = c;
    }
  }
  uint64_t l = 0;
  for (int lev = 22; lev <= 32; ++lev) {
    unsigned dig = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double c = __dmul_rn(0.5, __dadd_rn(lo[a], hi[a]));
      const bool up = x[a] >= c;
      lo[a] = up ? c : lo[a];
      hi[a] = up ? hi[a] : c;
      dig |= (unsigned)up << a;
    }
    l = (l << 3) | dig;
  }
  return l;
}

// key_lo of the built tree from its leaf-order points (downloads): sorted
// (skl) and by point index (kl)
template <typename R>
__global__ void __launch_bounds__(kNT) k_keys_lo_leaf(const V4<R>* squ, const int* perm, int64_t n,
                                                      const double* root, const uint64_t* skh,
                                                      uint64_t* skl, uint64_t* kl) {
  const int64_t t = blockIdx.x * (int64_t)kNT + threadIdx.x;
  if (t >= n) return;
  const V4<R> q = ld4(squ + t);
  const double x[3] = {(double)q.x, (double)q.y, (double)q.z};
  const uint64_t l = key_lo_of(x, skh[t], root);
  skl[t] = l;
  kl[perm[t]] = l;
}

// ------------------------------------------------------------ radix sort ---
// Stable LSD radix sort of (u64 key, i32 value), 8-bit digits, one-sweep
// passes (below): stable within-tile ranking with warp ballots/popc.
constexpr int kRsNT = 256;  // threads per tile; keys per thread (IPT) is a template parameter
constexpr int kHistWords = 7 * 512;  // digit histograms of every pass (8 x 256 or 7 x 512)


// ---- one-sweep passes ---------------------------------------------------------
// Digit histograms are independent of the key order, so ONE kernel counts every
// pass's digits up front (k0: p0 passes, then k1: p1 passes); each pass is then
// ONE kernel: a tile takes its id from an atomic counter (so every earlier tile
// has started), ranks its keys with warp ballots, publishes its per-digit
// count, and looks back over earlier tiles' published counts / inclusive
// prefixes (decoupled look-back, one 32-bit status word per tile and digit:
// flag << 30 | count) for its global offsets, then scatters. 1 launch per pass
// instead of 3, and no ntiles x 256 prefix pass.
constexpr unsigned kRsFlagAgg = 1u << 30, kRsFlagPrefix = 2u << 30, kRsCountMask = (1u << 30) - 1;

// digit histograms of all 8 passes in one read of the keys
template <int kRsIPT, int BITS = 8>
__global__ void __launch_bounds__(kRsNT) k_rs_hist_all(const uint64_t* key, int64_t n, unsigned* hist) {
  GS_PDL_ENTRY();
  constexpr int DIG = 1 << BITS, NP = (63 + BITS - 1) / BITS;
  __shared__ unsigned hs[NP * DIG];
  for (int t = threadIdx.x; t < NP * DIG; t += kRsNT) hs[t] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * (kRsNT * kRsIPT);
  for (int r = 0; r < kRsIPT; ++r) {
    const int64_t i = base + r * kRsNT + threadIdx.x;
    if (i >= n) break;
    const uint64_t k = key[i];
#pragma unroll
    for (int q = 0; q < NP; ++q) atomicAdd(&hs[q * DIG + ((unsigned)(k >> (BITS * q)) & (DIG - 1))], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < NP * DIG; t += kRsNT)
    if (hs[t]) atomicAdd(&hist[t], hs[t]);
}

// The lanes of the warp holding the same BITS-bit digit as this one (0 for
// !ok lanes, which are nobody's peers): one ballot per digit bit -- a lane's
// peers agree with it on every bit. Replaces MATCH.ANY, whose cost grows with
// the number of distinct values among the lanes (a third of a one-sweep
// pass's time at 1M with ~32 distinct digits per warp).
template <int BITS>
__device__ __forceinline__ unsigned peer_mask(unsigned d, bool ok) {
  unsigned pm = __ballot_sync(0xffffffffu, ok);
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const bool bit = (d >> b) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, bit);
    pm &= bit ? bal : ~bal;
  }
  return ok ? pm : 0u;
}

// NT threads x IPT keys per tile; the digit-parallel parts (scans, look-back)
// run on threads 0..255, one digit each. 256 x 8 (4 tiles per SM): N = 1M is
// one wave of 489 tiles; 512 x 8 (2 per SM) 245 tiles, 1024 x 8 (1 per SM)
// 123 -- each halving the look-back chain, the critical path of a pass (a
// tile finds its prefix ~tile / 16 round trips after the pass starts).
constexpr int kLB = 8;  // look-back: predecessors' status words loaded per round trip
template <int kRsIPT, int NT, int BITS = 8>
constexpr size_t onesweep_smem() {
  return sizeof(unsigned) * (NT / 32) * (1 << BITS) + sizeof(unsigned) * 2 * (1 << BITS) +
         sizeof(uint64_t) * NT * kRsIPT + sizeof(int) * NT * kRsIPT;
}
template <int kRsIPT, int NT, int BITS = 8>
__global__ void __launch_bounds__(NT, NT == 1024 ? 1 : (NT == 512 ? 2 : 4)) k_rs_onesweep(const uint64_t* kin, const int* vin,
                                                      uint64_t* kout, int* vout, int64_t n,
                                                      int shift, const unsigned* dig_tot,
                                                      unsigned* desc, unsigned* tile_ctr) {
  GS_PDL_ENTRY();
  constexpr int kTile = NT * kRsIPT;
  constexpr int DIG = 1 << BITS;
  constexpr unsigned kMask = DIG - 1;
  static_assert(NT >= DIG, "one digit per thread");
  extern __shared__ __align__(16) unsigned char os_smem[];
  // per-warp digit counts -> offsets within the tile's digit run; tile-local
  // digit starts; global position of tile-local slot 0 of each digit run; the
  // tile in digit order (coalesced write-out)
  unsigned (*wh)[DIG] = reinterpret_cast<unsigned (*)[DIG]>(os_smem);
  unsigned* ts = reinterpret_cast<unsigned*>(os_smem + sizeof(unsigned) * (NT / 32) * DIG);
  unsigned* gofs = ts + DIG;
  uint64_t* sk = reinterpret_cast<uint64_t*>(gofs + DIG);
  int* sv = reinterpret_cast<int*>(sk + kTile);
  __shared__ unsigned wsum[2][DIG / 32];  // per-warp sums of the two digit scans
  __shared__ int s_tile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool dig_thread = threadIdx.x < DIG;
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(tile_ctr, 1u);
  for (int i = threadIdx.x; i < (NT / 32) * DIG; i += NT) (&wh[0][0])[i] = 0;
  const unsigned dtot = dig_thread ? dig_tot[threadIdx.x] : 0u;
  __syncthreads();
  const int tile = s_tile;
  const int64_t t0 = (int64_t)tile * kTile;
  const int64_t seg = t0 + (int64_t)warp * (32 * kRsIPT);
  uint64_t key[kRsIPT];
  int val[kRsIPT];
  unsigned loc[kRsIPT];
  // all loads in flight before the first warp-synchronous digit match
#pragma unroll
  for (int r = 0; r < kRsIPT; ++r) {
    const int64_t i = seg + r * 32 + lane;
    const bool ok = i < n;
    key[r] = ok ? kin[i] : 0ull;
    val[r] = ok ? (vin ? vin[i] : (int)i) : 0;  // first pass: values are the indices
  }
  // per key: the lanes with the same digit (peer_mask); the group's leader
  // reserves cnt slots of the warp's digit counter with one shared atomic
  // (issued back to back for the kRsIPT keys: same-address atomics of one
  // warp stay in program order), lanes rank by lane order
  unsigned peers[kRsIPT], old[kRsIPT];
#pragma unroll
  for (int r = 0; r < kRsIPT; ++r) {
    const bool ok = seg + r * 32 + lane < n;
    const unsigned d = (unsigned)(key[r] >> shift) & kMask;
    // (invalid lanes -- tail tile only -- are nobody's peers)
    peers[r] = peer_mask<BITS>(d, ok);
  }
#pragma unroll
  for (int r = 0; r < kRsIPT; ++r) {
    const unsigned pm = peers[r];
    old[r] = 0;
    if (pm && lane == __ffs(pm) - 1)
      old[r] = atomicAdd(&wh[warp][(unsigned)(key[r] >> shift) & kMask], (unsigned)__popc(pm));
  }
#pragma unroll
  for (int r = 0; r < kRsIPT; ++r) {
    const unsigned pm = peers[r];
    const int leader = pm ? __ffs(pm) - 1 : lane;
    const unsigned base = __shfl_sync(0xffffffffu, old[r], leader);
    loc[r] = base + __popc(pm & ((1u << lane) - 1u));
  }
  __syncthreads();
  const unsigned d = threadIdx.x & kMask;
  unsigned tot = 0;
  if (dig_thread)
    for (int w = 0; w < NT / 32; ++w) {
      const unsigned t = wh[w][d];
      wh[w][d] = tot;
      tot += t;
    }
  // publish this tile's count for digit d as early as possible (look-back)
  cuda::atomic_ref<unsigned, cuda::thread_scope_device> mine(desc[(int64_t)tile * DIG + d]);
  if (dig_thread && tile != 0) mine.store(kRsFlagAgg | tot, cuda::memory_order_relaxed);
  // inclusive scans over digits (thread d = digit d): global digit totals and
  // this tile's counts -- warp shuffles, then the 8 warp sums
  unsigned gi = dtot, ti = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned g = __shfl_up_sync(0xffffffffu, gi, o), t = __shfl_up_sync(0xffffffffu, ti, o);
    if (lane >= o) gi += g, ti += t;
  }
  if (dig_thread && lane == 31) wsum[0][warp] = gi, wsum[1][warp] = ti;
  __syncthreads();
  if (dig_thread)
    for (int w = 0; w < warp; ++w) gi += wsum[0][w], ti += wsum[1][w];
  const unsigned tstart = ti - tot;
  // this tile's offset inside digit d: decoupled look-back over earlier tiles
  unsigned excl = 0;
  if (!dig_thread) {
  } else if (tile == 0) {
    mine.store(kRsFlagPrefix | tot, cuda::memory_order_relaxed);
  } else {
    // kLB predecessors' status words per round trip (independent loads),
    // consumed in order; an unpublished one is polled again from there
    for (int t = tile - 1;;) {
      unsigned v[kLB];
#pragma unroll
      for (int k = 0; k < kLB; ++k) {
        v[k] = kRsFlagPrefix;  // (before tile 0: never reached, tile 0 is a prefix)
        if (t - k >= 0) {
          cuda::atomic_ref<unsigned, cuda::thread_scope_device> prev(desc[(int64_t)(t - k) * DIG + d]);
          v[k] = prev.load(cuda::memory_order_relaxed);
        }
      }
      bool done = false;
      int used = 0;
#pragma unroll
      for (int k = 0; k < kLB; ++k) {
        if (done || used < k) break;  // stopped at a prefix or an unpublished tile
        if (!(v[k] & (kRsFlagAgg | kRsFlagPrefix))) break;  // that tile has not published yet
        excl += v[k] & kRsCountMask;
        ++used;
        if (v[k] & kRsFlagPrefix) done = true;
      }
      if (done) break;
      t -= used;
    }
    mine.store(kRsFlagPrefix | (excl + tot), cuda::memory_order_relaxed);
  }
  if (dig_thread) {
    gofs[d] = gi - dtot + excl - tstart;
    ts[d] = tstart;
  }
  __syncthreads();
  // stage the tile in (digit, rank) order ...
#pragma unroll
  for (int r = 0; r < kRsIPT; ++r) {
    if (seg + r * 32 + lane < n) {
      const unsigned dd = (unsigned)(key[r] >> shift) & kMask;
      const unsigned slot = ts[dd] + wh[warp][dd] + loc[r];
      sk[slot] = key[r];
      sv[slot] = val[r];
    }
  }
  __syncthreads();
  // ... and write it out: consecutive slots of one digit run are consecutive
  // output positions (coalesced), instead of 12-B scatters per key
  const int cnt = n - t0 < kTile ? (int)(n - t0) : kTile;
#pragma unroll
  for (int r = 0; r < kRsIPT; ++r) {
    const int i = r * NT + threadIdx.x;
    if (i < cnt) {
      const uint64_t k = sk[i];
      const unsigned pos = gofs[(unsigned)(k >> shift) & kMask] + (unsigned)i;
      kout[pos] = k;
      vout[pos] = sv[i];
    }
  }
}

// one one-sweep pass, IPT keys per thread
int onesweep(int ipt, int nt, int ntiles, cudaStream_t st, const uint64_t* ki, const int* vi,
             uint64_t* ko, int* vo, int64_t n, int shift, const unsigned* dig_tot, unsigned* desc,
             unsigned* ctr, int bits = 8) {
  if (nt == 1024 && bits == 9) {
    static const bool attr = [] {
      cudaFuncSetAttribute(k_rs_onesweep<8, 1024, 9>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)onesweep_smem<8, 1024, 9>());
      return true;
    }();
    (void)attr;
    GS_CUDA_OK(pdl_launch(k_rs_onesweep<8, 1024, 9>, ntiles, 1024, onesweep_smem<8, 1024, 9>(), st, ki, vi, ko, vo, n, shift, dig_tot, desc, ctr));
  } else if (nt == 1024) {
    static const bool attr = [] {
      cudaFuncSetAttribute(k_rs_onesweep<8, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)onesweep_smem<8, 1024>());
      return true;
    }();
    (void)attr;
    GS_CUDA_OK(pdl_launch(k_rs_onesweep<8, 1024>, ntiles, 1024, onesweep_smem<8, 1024>(), st, ki, vi, ko, vo, n, shift, dig_tot, desc, ctr));
  } else if (nt == 512) {
    static const bool attr = [] {
      cudaFuncSetAttribute(k_rs_onesweep<8, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)onesweep_smem<8, 512>());
      return true;
    }();
    (void)attr;
    GS_CUDA_OK(pdl_launch(k_rs_onesweep<8, 512>, ntiles, 512, onesweep_smem<8, 512>(), st, ki, vi, ko, vo, n, shift, dig_tot, desc, ctr));
  } else if (ipt == 8) {
    GS_CUDA_OK(pdl_launch(k_rs_onesweep<8, 256>, ntiles, 256, onesweep_smem<8, 256>(), st, ki, vi, ko, vo, n, shift, dig_tot, desc, ctr));
  } else {
    GS_CUDA_OK(pdl_launch(k_rs_onesweep<4, 256>, ntiles, 256, onesweep_smem<4, 256>(), st, ki, vi, ko, vo, n, shift, dig_tot, desc, ctr));
  }
  return GS_OK;
}

// ---------------------------------------------------------------- ties ---
// Points sharing all 21 levels of key_hi form runs of equal keys in the
// key_hi-sorted order (the sort is stable: a run is in ascending index). The
// full order sorts each run stably by key_lo (levels 22-32), computed for the
// run members only and carried with the index as the 64-bit code
// (key_lo << 31) | index. k_tie_runs lists the runs (and sets the tie flag);
// k_tie_sort, one cooperative grid, sorts them in place:
//  * a run of <= 64 points: a warp, rank by comparison;
//  * a run of <= 2048 points: a CTA, bitonic sort in shared memory;
//  * longer runs (a diverged flow whose root box dwarfs the cloud -- config
//    4's puts 77 % of the points in such runs): a segmented LSD radix sort of
//    key_lo, 5 passes of 8 bits over 2048-point chunks spread across the
//    grid: per-chunk digit counts, per-run offsets (run-local, digit-major),
//    stable scatter (warp match.any ranking: run keys share most digits, few
//    distinct values per warp) -- each pass
//    three grid.sync()s apart.
// Two launches whatever the data, and no no-op passes when there is no tie.
namespace cg = cooperative_groups;
constexpr int kTieChunk = 2048;
constexpr int kTieSmallCtr = 28, kTieBigCtr = 29, kTieFlag = 31;  // sort counters
constexpr int kScanTicket = 27;

// L[t] = common digits of sorted neighbours t, t + 1 from key_hi (21 where
// they tie: k_tie_sort completes those from key_lo), and the runs listed
__global__ void k_lcp_runs(const uint64_t* skh, int64_t n, int* L, unsigned* ctr, int2* small_runs,
                           int4* big_runs) {
  GS_PDL_ENTRY();
  const int64_t t = blockIdx.x * (int64_t)kNT + threadIdx.x;
  if (t + 1 >= n) return;
  const uint64_t k = skh[t], k1 = skh[t + 1];
  const uint64_t x = k ^ k1;
  L[t] = x ? (__clzll((long long)x) - 1) / 3 : 21;
  if (k1 != k || (t > 0 && skh[t - 1] == k)) return;  // not a run start
  // last index of the run: exponential then binary search on equality
  int64_t step = 1, good = t + 1;
  while (good + step < n && skh[good + step] == k) {
    good += step;
    step <<= 1;
  }
  int64_t lo = good, hi = min(n - 1, good + step);
  while (hi > lo) {
    const int64_t mid = lo + (hi - lo + 1) / 2;
    if (skh[mid] == k) lo = mid;
    else hi = mid - 1;
  }
  const int len = (int)(lo - t + 1);
  if (len <= 64) small_runs[atomicAdd(ctr + kTieSmallCtr, 1u)] = make_int2((int)t, len);
  else big_runs[atomicAdd(ctr + kTieBigCtr, 1u)] = make_int4((int)t, len, 0, 0);
  atomicOr(ctr + kTieFlag, 1u);
}

// (key_lo << 31) | index: unique per point (n < 2^31), ordered as the full key
// key_lo source of the tie sort: k_keys' array, or a replay from the point
struct TieKeys {
  const uint64_t* klo;
  const void* rec;  // the build's records (float4 / double4 pairs)
  const double* root;
  const uint64_t* skh;
  int f32;
  int valid;  // k_keys computed klo this build
};
__device__ __forceinline__ uint64_t tie_code(const TieKeys& tk, const int* perm, int64_t j) {
  const int p = perm[j];
  uint64_t l;
  if (tk.valid) {
    l = tk.klo[p];
  } else {
    double x[3];
    if (tk.f32) {
      const float4 q = ld4(static_cast<const float4*>(tk.rec) + 2 * (int64_t)p);
      x[0] = q.x; x[1] = q.y; x[2] = q.z;
    } else {
      const double4 q = ld4(static_cast<const double4*>(tk.rec) + 2 * (int64_t)p);
      x[0] = q.x; x[1] = q.y; x[2] = q.z;
    }
    l = key_lo_of(x, tk.skh[j], tk.root);
  }
  return (l << 31) | (uint64_t)p;
}

__device__ __forceinline__ void tie_put(int* perm, uint64_t* skl, int64_t j, uint64_t c) {
  perm[j] = (int)(c & 0x7fffffffu);
  skl[j] = c >> 31;
}

// common digits of two tied neighbours (equal key_hi) from their codes
__device__ __forceinline__ int tie_lcp(uint64_t ca, uint64_t cb) {
  const uint64_t y = (ca ^ cb) >> 31;
  return y ? 21 + (__clzll((long long)y) - 31) / 3 : 32;
}

// bitonic sort of s[0, P) (P a power of two) by the CTA
__device__ void bitonic_smem(uint64_t* s, int P) {
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int ij = i ^ j;
        if (ij > i) {
          const uint64_t u = s[i], v = s[ij];
          if ((u > v) == ((i & k) == 0)) {
            s[i] = v;
            s[ij] = u;
          }
        }
      }
      __syncthreads();
    }
}

// exclusive prefix of f(run) over the long-run list by CTA 0 (block scan in
// rounds of kNT runs); writes it through put(run, prefix), returns the total
template <typename F, typename P>
__device__ int tie_prefix(int nbig, F f, P put) {
  __shared__ int s_carry;
  __shared__ int ws[kNT / 32];
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nbig; b0 += kNT) {
    const int r = b0 + threadIdx.x;
    const int c = r < nbig ? f(r) : 0;
    int v = c;
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane == 31) ws[threadIdx.x >> 5] = v;
    __syncthreads();
    int add = s_carry;
    for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) add += ws[w];
    if (r < nbig) put(r, add + v - c);
    __syncthreads();
    if (threadIdx.x == kNT - 1) s_carry = add + v;
    __syncthreads();
  }
  return s_carry;
}

// task g -> the run whose task prefix (field F of the list) covers it
template <int F>
__device__ __forceinline__ int tie_task_run(const int4* big, int nbig, int g) {
  int lo = 0, hi = nbig - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if ((F == 2 ? big[mid].z : big[mid].w) <= g) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

constexpr int kTieGroup = 16;  // chunks per digit-count group (look-up of a chunk's offsets)

__global__ void __launch_bounds__(kNT) k_tie_sort(TieKeys klo, const unsigned* lo_valid,
                                                  const unsigned* ctr,
                                                  const int2* small_runs, int4* big_runs,
                                                  int* perm, uint64_t* skl, uint64_t* bufa,
                                                  uint64_t* bufb, unsigned* scr, int* L) {
  GS_PDL_ENTRY();
  if (ctr[kTieFlag] == 0) return;  // (uniform over the grid)
  klo.valid = (int)*lo_valid;
  cg::grid_group grid = cg::this_grid();
  __shared__ uint64_t s[kTieChunk];
  __shared__ unsigned wh[kNT / 32][256];
  __shared__ unsigned soff[256];
  __shared__ unsigned ws[kNT / 32];
  __shared__ int s_nt[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // runs of <= 64 points: a warp each
  const int nsmall = (int)ctr[kTieSmallCtr];
  const int gw = (blockIdx.x * kNT + threadIdx.x) >> 5, nw = (gridDim.x * kNT) >> 5;
  for (int r = gw; r < nsmall; r += nw) {
    const int2 run = small_runs[r];
    // two codes per lane (runs of <= 64): rank = number of smaller codes
    const uint64_t c0 = lane < run.y ? tie_code(klo, perm, (int64_t)run.x + lane) : ~0ull;
    const uint64_t c1 = lane + 32 < run.y ? tie_code(klo, perm, (int64_t)run.x + 32 + lane) : ~0ull;
    int r0 = 0, r1 = 0;
    for (int k = 0; k < min(run.y, 32); ++k) {
      const uint64_t u = __shfl_sync(0xffffffffu, c0, k);
      r0 += u < c0;
      r1 += u < c1;
    }
    for (int k = 32; k < run.y; ++k) {
      const uint64_t u = __shfl_sync(0xffffffffu, c1, k - 32);
      r0 += u < c0;
      r1 += u < c1;
    }
    __syncwarp();
    if (lane < run.y) tie_put(perm, skl, (int64_t)run.x + r0, c0);
    if (lane + 32 < run.y) tie_put(perm, skl, (int64_t)run.x + r1, c1);
    // the run's internal neighbour lcps: each code's successor in the order
    // is the smallest larger code
    uint64_t n0 = ~0ull, n1 = ~0ull;
    for (int k = 0; k < run.y; ++k) {
      const uint64_t u = __shfl_sync(0xffffffffu, k < 32 ? c0 : c1, k & 31);
      if (u > c0 && u < n0) n0 = u;
      if (u > c1 && u < n1) n1 = u;
    }
    if (lane < run.y && r0 + 1 < run.y) L[run.x + r0] = tie_lcp(c0, n0);
    if (lane + 32 < run.y && r1 + 1 < run.y) L[run.x + r1] = tie_lcp(c1, n1);
  }
  const int nbig = (int)ctr[kTieBigCtr];
  if (nbig == 0) return;
  // task numbering (CTA 0): .z = chunk prefix over all long runs (phase A);
  // .w = slot prefix of the multi-chunk runs' chunks, each run padded to
  // whole groups of kTieGroup slots; totals in the sentinel big_runs[nbig]
  if (blockIdx.x == 0) {
    const int ta = tie_prefix(nbig, [&](int r) { return (big_runs[r].y + kTieChunk - 1) / kTieChunk; },
                              [&](int r, int v) { big_runs[r].z = v; });
    const int tb = tie_prefix(nbig, [&](int r) {
      const int L = big_runs[r].y;
      const int nc = (L + kTieChunk - 1) / kTieChunk;
      return L > kTieChunk ? (nc + kTieGroup - 1) / kTieGroup * kTieGroup : 0; },
      [&](int r, int v) { big_runs[r].w = v; });
    if (threadIdx.x == 0) big_runs[nbig] = make_int4(0, 0, ta, tb);
  }
  grid.sync();
  if (threadIdx.x == 0) {
    const int4 tot = big_runs[nbig];
    s_nt[0] = tot.z;
    s_nt[1] = tot.w;
  }
  __syncthreads();
  const int na = s_nt[0], nm = s_nt[1];  // nm: slots (a multiple of kTieGroup)
  const int ngrp = nm / kTieGroup;
  // scratch: per-slot digit counts [nm][256], per-group sums [2][ngrp][256]
  unsigned* chist = scr;
  unsigned* gsum = scr + (size_t)nm * 256;
  // phase A: codes; a single-chunk run is sorted (bitonic) and finished here
  for (int g = blockIdx.x; g < na; g += gridDim.x) {
    const int4 run = big_runs[tie_task_run<2>(big_runs, nbig, g)];
    const int c0 = (g - run.z) * kTieChunk, cl = min(kTieChunk, run.y - c0);
    if (run.y > kTieChunk) {
      for (int i = threadIdx.x; i < cl; i += kNT)
        bufa[(int64_t)run.x + c0 + i] = tie_code(klo, perm, (int64_t)run.x + c0 + i);
      continue;
    }
    int P = 1;
    while (P < cl) P <<= 1;
    for (int i = threadIdx.x; i < P; i += kNT)
      s[i] = i < cl ? tie_code(klo, perm, (int64_t)run.x + i) : ~0ull;
    __syncthreads();
    bitonic_smem(s, P);
    for (int i = threadIdx.x; i < cl; i += kNT) {
      tie_put(perm, skl, (int64_t)run.x + i, s[i]);
      if (i + 1 < cl) L[run.x + i] = tie_lcp(s[i], s[i + 1]);
    }
    __syncthreads();
  }
  if (nm == 0) return;  // (uniform)
  // this CTA's slots g = blockIdx.x + k gridDim.x: their runs, looked up once
  __shared__ int s_run[64];
  for (int k = threadIdx.x; k < 64; k += kNT) {
    const int g = blockIdx.x + k * gridDim.x;
    s_run[k] = g < nm ? tie_task_run<3>(big_runs, nbig, g) : 0;
  }
  __syncthreads();
  auto run_of = [&](int g) {
    const int k = (g - (int)blockIdx.x) / (int)gridDim.x;
    return k < 64 ? s_run[k] : tie_task_run<3>(big_runs, nbig, g);
  };
  for (int64_t k = blockIdx.x * (int64_t)kNT + threadIdx.x; k < (int64_t)ngrp * 256;
       k += (int64_t)gridDim.x * kNT)
    gsum[k] = 0;
  // segmented LSD radix passes over key_lo (code bits 31..63), two
  // grid-synchronised phases each: digit counts, then offsets + scatter
  constexpr int kIPT = kTieChunk / kNT;  // 8 codes per thread: element 256 w + 32 r + lane
  uint64_t* src = bufa;
  uint64_t* dst = bufb;
  for (int pass = 0; pass < 5; ++pass) {
    const int shift = 31 + 8 * pass;
    unsigned* gs = gsum + (size_t)(pass & 1) * ngrp * 256;
    unsigned* gnext = gsum + (size_t)((pass + 1) & 1) * ngrp * 256;
    grid.sync();
    // (1) digit counts per chunk, summed per group; the next pass's group sums zeroed
    for (int g = blockIdx.x; g < nm; g += gridDim.x) {
      const int r = run_of(g);
      const int4 run = big_runs[r];
      const int c0 = (g - run.w) * kTieChunk;
      if (c0 >= run.y) continue;  // a padding slot (uniform)
      const int cl = min(kTieChunk, run.y - c0);
      unsigned* hs = &wh[0][0];
      hs[threadIdx.x] = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < cl; i += kNT)
        atomicAdd(&hs[(unsigned)(src[(int64_t)run.x + c0 + i] >> shift) & 255u], 1u);
      __syncthreads();
      const unsigned v = hs[threadIdx.x];
      chist[(size_t)g * 256 + threadIdx.x] = v;
      if (v) atomicAdd(&gs[(size_t)(g / kTieGroup) * 256 + threadIdx.x], v);
      __syncthreads();
    }
    for (int64_t k = blockIdx.x * (int64_t)kNT + threadIdx.x; k < (int64_t)ngrp * 256;
         k += (int64_t)gridDim.x * kNT)
      gnext[k] = 0;
    grid.sync();
    // (2) each chunk: run-local digit starts (scan of the run's group sums),
    // its offset within each digit (earlier groups + earlier chunks of its
    // group), then the stable scatter
    for (int g = blockIdx.x; g < nm; g += gridDim.x) {
      const int r = run_of(g);
      const int4 run = big_runs[r];
      const int c0 = (g - run.w) * kTieChunk;
      if (c0 >= run.y) continue;
      const int cl = min(kTieChunk, run.y - c0);
      const int nc = (run.y + kTieChunk - 1) / kTieChunk;
      const int G0 = run.w / kTieGroup, G1 = G0 + (nc + kTieGroup - 1) / kTieGroup, G = g / kTieGroup;
      {
        const unsigned d = threadIdx.x;
        unsigned tot = 0, pre = 0;
#pragma unroll 8
        for (int q = G0; q < G1; ++q) {
          const unsigned x = __ldcg(gs + (size_t)q * 256 + d);
          tot += x;
          pre += q < G ? x : 0u;
        }
#pragma unroll 8
        for (int c = G * kTieGroup; c < g; ++c) pre += __ldcg(chist + (size_t)c * 256 + d);
        unsigned v = tot;  // exclusive scan over the 256 digits
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned u = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += u;
        }
        if (lane == 31) ws[warp] = v;
        __syncthreads();
        unsigned base = v - tot;
        for (int w = 0; w < warp; ++w) base += ws[w];
        soff[d] = base + pre;
      }
      for (int w = 0; w < kNT / 32; ++w) wh[w][threadIdx.x] = 0;
      __syncthreads();
      uint64_t key[kIPT];
      unsigned loc[kIPT];
#pragma unroll
      for (int q = 0; q < kIPT; ++q) {
        const int i = warp * 32 * kIPT + q * 32 + lane;
        key[q] = i < cl ? __ldcg(src + (int64_t)run.x + c0 + i) : 0ull;
      }
#pragma unroll
      for (int q = 0; q < kIPT; ++q) {
        const int i = warp * 32 * kIPT + q * 32 + lane;
        const bool ok = i < cl;
        const unsigned dg = (unsigned)(key[q] >> shift) & 255u;
        const unsigned pm = __match_any_sync(0xffffffffu, ok ? dg : 256u);
        unsigned old = 0;
        if (ok && lane == __ffs(pm) - 1) old = atomicAdd(&wh[warp][dg], (unsigned)__popc(pm));
        const unsigned b = __shfl_sync(0xffffffffu, old, __ffs(pm) - 1);
        loc[q] = b + __popc(pm & ((1u << lane) - 1u));
      }
      __syncthreads();
      {  // warp offsets within the chunk's digit runs
        const unsigned d = threadIdx.x;
        unsigned acc = 0;
        for (int w = 0; w < kNT / 32; ++w) {
          const unsigned x = wh[w][d];
          wh[w][d] = acc;
          acc += x;
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kIPT; ++q) {
        const int i = warp * 32 * kIPT + q * 32 + lane;
        if (i < cl) {
          const unsigned dg = (unsigned)(key[q] >> shift) & 255u;
          dst[(int64_t)run.x + soff[dg] + wh[warp][dg] + loc[q]] = key[q];
        }
      }
      __syncthreads();
    }
    uint64_t* t = src;
    src = dst;
    dst = t;
  }
  grid.sync();
  for (int g = blockIdx.x; g < nm; g += gridDim.x) {
    const int4 run = big_runs[run_of(g)];
    const int c0 = (g - run.w) * kTieChunk;
    if (c0 >= run.y) continue;
    const int cl = min(kTieChunk, run.y - c0);
    for (int i = threadIdx.x; i < cl; i += kNT) {
      const int64_t j = (int64_t)run.x + c0 + i;
      const uint64_t c = __ldcg(src + j);
      tie_put(perm, skl, j, c);
      if (c0 + i + 1 < run.y) L[j] = tie_lcp(c, __ldcg(src + j + 1));
    }
  }
}

// ------------------------------------------------------------- topology ---


__device__ __forceinline__ int lm_of(const int* L, int64_t a) { return a > 0 ? L[a - 1] : -1; }


// nodes starting at position a: internal levels (Lm, min(Lp,31)] + one leaf
// unless a continues a depth-32 bucket.
__device__ __forceinline__ void starts(const int* L, int64_t n, int64_t a, int& Lm, int& Lp,
                                       int& cint, int& leaf) {
  Lm = lm_of(L, a);
  Lp = a + 1 < n ? L[a] : -1;
  cint = max(0, min(Lp, 31) - Lm);
  leaf = Lm < 32 ? 1 : 0;
}


// lcp(a, x) >= l from the sorted keys. Levels <= 21 need key_hi only (one
// 8-B load per probe); deeper levels exist only where neighbours tie and also
// compare key_lo. Two instantiations, so the common search carries no key_lo
// code at all (a merged version executed the deep branch predicated off: 12 %
// of the node table's instructions).
template <bool DEEP>
__device__ __forceinline__ bool prefix_ge(uint64_t ah, uint64_t al, const uint64_t* kh,
                                          const uint64_t* kl, int64_t x, int l) {
  const uint64_t bh = kh[x];
  if (!DEEP) return ((ah ^ bh) >> (3 * (21 - l))) == 0;
  if (ah != bh) return false;
  return ((al ^ kl[x]) >> (3 * (32 - l))) == 0;
}

// largest b >= a with lcp(a, b) >= l
template <bool DEEP>
__device__ int64_t search_right_t(const uint64_t* kh, const uint64_t* kl, int64_t n, int64_t a,
                                  int l) {
  const uint64_t ah = kh[a], al = DEEP ? kl[a] : 0;
  int64_t step = 1, good = a;
  while (a + step < n && prefix_ge<DEEP>(ah, al, kh, kl, a + step, l)) {
    good = a + step;
    step <<= 1;
  }
  int64_t lo = good, hi = min(n - 1, a + step);  // lo good, (hi bad or end)
  while (hi > lo) {
    const int64_t mid = lo + (hi - lo + 1) / 2;
    if (prefix_ge<DEEP>(ah, al, kh, kl, mid, l)) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}
__device__ __forceinline__ int64_t search_right(const uint64_t* kh, const uint64_t* kl, int64_t n,
                                                int64_t a, int l) {
  return l > 21 ? search_right_t<true>(kh, kl, n, a, l) : search_right_t<false>(kh, kl, n, a, l);
}

// smallest s <= a with lcp(s, a) >= l
template <bool DEEP>
__device__ int64_t search_left_t(const uint64_t* kh, const uint64_t* kl, int64_t a, int l) {
  const uint64_t ah = kh[a], al = DEEP ? kl[a] : 0;
  int64_t step = 1, good = a;
  while (a - step >= 0 && prefix_ge<DEEP>(ah, al, kh, kl, a - step, l)) {
    good = a - step;
    step <<= 1;
  }
  int64_t hi = good, lo = max((int64_t)0, a - step);
  while (hi > lo) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (prefix_ge<DEEP>(ah, al, kh, kl, mid, l)) hi = mid;
    else lo = mid + 1;
  }
  return hi;
}
__device__ __forceinline__ int64_t search_left(const uint64_t* kh, const uint64_t* kl, int64_t a,
                                               int l) {
  return l > 21 ? search_left_t<true>(kh, kl, a, l) : search_left_t<false>(kh, kl, a, l);
}

__device__ int parent_of(const uint64_t* kh, const uint64_t* kl, const int* L, const int* first,
                         int64_t a, int plevel) {
  const int64_t s = search_left(kh, kl, a, plevel);
  return first[s] + (plevel - (lm_of(L, s) + 1));
}

// The start position of every node: position a starts nodes
// [first[a], first[a + 1]) -- cheap writes, so the searches below run one
// node per thread (a position starting many levels no longer serialises them).
__global__ void k_node_starts(const int* first, int64_t n, int64_t cap, int* start,
                              int* overflow) {
  GS_PDL_ENTRY();
  const int64_t a = blockIdx.x * (int64_t)kNT + threadIdx.x;
  if (a >= n) return;
  if (first[n] > cap) {  // more nodes than the arrays hold (degenerate clustering)
    if (a == 0 && overflow) atomicExch(overflow, 1);
    return;
  }
  for (int idx = first[a]; idx < first[a + 1]; ++idx) start[idx] = (int)a;
}

// One node per thread: node idx starts at a = start[idx]; it is internal
// node k = idx - first[a] of the levels L[a-1]+1 .. min(L[a], 31) starting
// there, or a's leaf (last). Its range end b is the last position whose key
// shares the node's level-l prefix (exponential + binary search on the sorted
// keys); its parent is the node above it at the same start, or -- for the
// first node at a position -- the level-(l-1) node found by a left search.
// inner[idx] = 1: internal node idx has an internal child (else it is a twig:
// all children leaves -- the flag the traversal records carry). Children are
// the maximal runs of its positions with lcp >= l + 1, so at level l < 31 it is
// a twig iff every neighbour lcp inside its range is exactly l (<= 8 points);
// at level 31 every child is a leaf. Parents (read by downloads only) are
// computed when want_parent: the node above at the same start, or -- for the
// first node at a position -- the level-(l-1) node found by a left search.
__global__ void k_nodes(const uint64_t* kh, const uint64_t* kl, const int* L, const int* first,
                        const int* start, int64_t n, int64_t cap, int4* meta, int* parent,
                        int* inner, int want_parent) {
  GS_PDL_ENTRY();
  const int64_t idx = blockIdx.x * (int64_t)kNT + threadIdx.x;
  const int m = first[n];
  if (m > cap || idx >= m) return;
  const int64_t a = start[idx];
  int Lm, Lp, ci, lf;
  starts(L, n, a, Lm, Lp, ci, lf);
  const int k = (int)(idx - first[a]);
  const int l0 = Lm + 1;
  if (k < ci) {  // internal node of level l0 + k
    const int l = l0 + k;
    const int64_t b = search_right(kh, kl, n, a, l);
    meta[idx] = make_int4(first[b + 1], (int)a, (int)b, l << 8);
    bool twig = l == 31;
    if (!twig && b - a < 8) {
      twig = true;
      for (int64_t t = a; t < b; ++t) twig = twig && L[t] == l;
    }
    inner[idx] = twig ? 0 : 1;
    if (want_parent)
      parent[idx] = l == 0 ? -1 : (k > 0 ? (int)idx - 1 : parent_of(kh, kl, L, first, a, l - 1));
    return;
  }
  int level;
  int64_t b = a;
  if (Lp == 32) {
    level = 32;
    b = search_right(kh, kl, n, a, 32);
  } else {
    level = max(Lm, Lp) + 1;
  }
  meta[idx] = make_int4(first[b + 1], (int)a, (int)b, (level << 8) | 1);
  inner[idx] = 0;
  if (want_parent)
    parent[idx] = level == 0 ? -1 : (level - 1 >= l0 ? (int)idx - 1 : parent_of(kh, kl, L, first, a, level - 1));
}

// per node: child count (the twig flag of the traversal record)

// ------------------------------------------------------------ aggregates ---
// Forward: tight AABB + sums of q and p; backward: sums of alpha and beta.
// Leaves sum their points in leaf order; an internal node is completed by the
// last child to arrive (atomic counter) as the sum of its children in child
// order -- deterministic whatever the arrival order.
template <typename R>
__global__ void __launch_bounds__(kNT) k_gather(const V4<R>* rec, const int* perm, int64_t n,
                                                double kap, double c0x, double c0y, double c0z,
                                                int scaled, V4<R>* srec, V4<R>* squ) {
  GS_PDL_ENTRY();
  const int64_t t = blockIdx.x * (int64_t)kNT + threadIdx.x;
  if (t >= n) return;
  const int i = perm[t];
  const V4<R> q = ld4(rec + 2 * i), p = ld4(rec + 2 * i + 1);
  st4(squ + t, q);
  V4<R> qs = q;
  if (scaled) {  // FP32 interaction coordinates, same rounding as the all-pairs path
    const float kf = (float)kap;
    qs = mk4<R>((R)fmaf(kf, (float)q.x, -(float)(kap * c0x)), (R)fmaf(kf, (float)q.y, -(float)(kap * c0y)),
                (R)fmaf(kf, (float)q.z, -(float)(kap * c0z)));
  }
  st4(srec + 2 * t, qs);
  st4(srec + 2 * t + 1, p);
}

template <typename R>
__global__ void k_gather_adj(const V4<R>* adj, const int* perm, int64_t n, V4<R>* sadj) {
  const int64_t t = blockIdx.x * (int64_t)kNT + threadIdx.x;
  if (t >= n) return;
  const int i = perm[t];
  st4(sadj + 2 * t, ld4(adj + 2 * i));
  st4(sadj + 2 * t + 1, ld4(adj + 2 * i + 1));
}

// ------------------------------------------------------------ aggregates ---
// Node aggregates (tight AABB + FP64 sums of q and p: mode 0; FP64 sums of
// alpha and beta: mode 1) and the traversal records, after k_nodes. The
// leaf order is cut into chunks of C points (256 up to 256k points, else
// 1024 FP32 / 512 FP64), one CTA
// each (k_agg_chunk). The CTA gathers its chunk's points (by perm, writing the
// leaf-order copies srec / squ or sadj on the way -- the build's gather fused
// in) into shared memory. The nodes that start in the chunk are a contiguous
// pre-order range [first[c0], first[c1]); those lying inside the chunk are
// summed from shared memory in range order (small ones by a thread, larger by
// a warp) and their records written. A node spanning chunks ("outer") is
// split at the chunk boundaries: its TAIL in its first chunk, whole chunks,
// its HEAD in its last chunk. Per level at most one outer node starts in a
// chunk and at most one (the one containing the chunk's first point) ends in
// it, so the CTA computes, from shared memory, its chunk's total and the tail
// and head ranges of every level (heads found from the lcp array: the level-l
// node containing the chunk's first point ends at the first position whose
// lcp with the next is < l). k_agg_outer then sums each outer node as tail +
// chunk totals + head, in chunk order. Every reduction order is fixed
// (deterministic), every point is read from HBM once per aggregate, and no
// kernel waits on another's partial results.
constexpr int kSmallNode = 16;  // inside nodes above this are summed by a warp
constexpr int kLevels = 33;     // levels 0..32 (32: depth-32 buckets)
constexpr int kPartPerChunk = 1 + 2 * kLevels;  // total, head[33], tail[33]

__device__ __forceinline__ float ival(float, int v) { return __int_as_float(v); }
__device__ __forceinline__ double ival(double, int v) { return (double)v; }

__device__ __forceinline__ double4 ldcg4(const double4* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldcg(q), b = __ldcg(q + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ float4 ldcg4(const float4* p) { return __ldcg(p); }

__device__ __forceinline__ bool is_single(const int4& mi) { return (mi.w & 1) && mi.y == mi.z; }


template <typename R>
struct AggArgs {
  const int4* meta;
  const int* nchild;
  const int* first;  // [n + 1] pre-order index of the first node starting at each position
  const int* lcp;    // [n - 1] common digits of leaf-order neighbours
  const int* perm;
  int64_t n;
  const V4<R>* rec;  // by point index: records (q, p) in mode 0, adjoints (alpha, beta) in mode 1
  V4<R>*srec, *squ, *sadj;  // leaf-order copies written on the way
  V4<R>*lo, *hi;
  double4 *s0, *s1;
  V4<R>*nrec, *nadj;
  // per chunk: total, head[level], tail[level] partial aggregates
  double4 *ps0, *ps1;
  V4<R>*plo, *phi;
  int* outer;      // outer nodes (listed by the chunk they start in)
  int* outer_big;  // outer nodes spanning > kBigSpan chunks (a CTA each in k_agg_outer)
  int* outer_cnt;  // [0] outer, [1] outer_big
  double kap, c0x, c0y, c0z;
  int scaled;
  int full;  // write the FP64 sums and boxes too (DevTree::lean = false)
};

// FP32 interaction coordinates, same rounding as the all-pairs path
template <typename R>
__device__ __forceinline__ V4<R> scaled_q(const AggArgs<R>& a, const V4<R>& q) {
  if (!a.scaled) return mk4<R>(q.x, q.y, q.z);
  const float kf = (float)a.kap;
  return mk4<R>((R)fmaf(kf, (float)q.x, -(float)(a.kap * a.c0x)),
                (R)fmaf(kf, (float)q.y, -(float)(a.kap * a.c0y)),
                (R)fmaf(kf, (float)q.z, -(float)(a.kap * a.c0z)));
}

struct Sums {
  double a[3], b[3];
};
template <typename R>
struct Box {
  R l[3], h[3];
};

template <typename R>
__device__ __forceinline__ void box_init(Box<R>& x) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    x.l[k] = R(INFINITY);
    x.h[k] = -R(INFINITY);
  }
}

template <typename R>
__device__ __forceinline__ void add_point(Sums& s, Box<R>& x, const V4<R>& u, const V4<R>& v, bool box) {
  s.a[0] += u.x; s.a[1] += u.y; s.a[2] += u.z;
  s.b[0] += v.x; s.b[1] += v.y; s.b[2] += v.z;
  if (box) {
    x.l[0] = min(x.l[0], u.x); x.l[1] = min(x.l[1], u.y); x.l[2] = min(x.l[2], u.z);
    x.h[0] = max(x.h[0], u.x); x.h[1] = max(x.h[1], u.y); x.h[2] = max(x.h[2], u.z);
  }
}

template <typename R>
__device__ __forceinline__ void add_part(Sums& s, Box<R>& x, const double4& d0, const double4& d1,
                                         const V4<R>& l, const V4<R>& h) {
  s.a[0] += d0.x; s.a[1] += d0.y; s.a[2] += d0.z;
  s.b[0] += d1.x; s.b[1] += d1.y; s.b[2] += d1.z;
  x.l[0] = min(x.l[0], l.x); x.l[1] = min(x.l[1], l.y); x.l[2] = min(x.l[2], l.z);
  x.h[0] = max(x.h[0], h.x); x.h[1] = max(x.h[1], h.y); x.h[2] = max(x.h[2], h.z);
}

// The traversal record of node i (mode 0) -- {centroid | point, code}
// {momentum sum | p, begin} {lo, count} {hi}, code = skip | single << 31 |
// bucket << 30 | twig << 29 (skip < 2^29) -- or its adjoint unit (mode 1)
// {alpha sum, beta mean}; plus the FP64 sums and the box of a non-single node.
// u, v: a single node's own point (q unscaled, p) / (alpha, beta).
template <typename R, int MODE>
__device__ void write_node(const AggArgs<R>& a, int i, const int4& mi, int nch, const Sums& s,
                           const Box<R>& x, const V4<R>& u, const V4<R>& v) {
  const int cnt = mi.z - mi.y + 1;
  const bool single = is_single(mi);
  if (MODE == 1) {
    if (single) {
      st4(a.nadj + 2 * i, mk4<R>(u.x, u.y, u.z));
      st4(a.nadj + 2 * i + 1, mk4<R>(v.x, v.y, v.z));
      return;
    }
    const double inv = 1.0 / cnt;
    st4(a.nadj + 2 * i, mk4<R>(R(s.a[0]), R(s.a[1]), R(s.a[2])));
    // db = beta_i - (1 / count) * beta_sum, bh_kernel.cpp:146
    st4(a.nadj + 2 * i + 1, mk4<R>(R(__dmul_rn(inv, s.b[0])), R(__dmul_rn(inv, s.b[1])),
                                   R(__dmul_rn(inv, s.b[2]))));
    if (a.full) {
      a.s0[i] = make_double4(s.a[0], s.a[1], s.a[2], 0.0);
      a.s1[i] = make_double4(s.b[0], s.b[1], s.b[2], 0.0);
    }
    return;
  }
  const bool leaf = mi.w & 1;
  // twig: an internal node whose children are all leaves (subtree = itself +
  // its children); opening it makes every point of it direct, no child gated
  const bool twig = !leaf && nch == 0;  // nch: has an internal child (k_nodes)
  const int code = mi.x | (single ? (int)0x80000000u : 0) | ((leaf && cnt > 1) ? 0x40000000 : 0) |
                   (twig ? 0x20000000 : 0);
  V4<R> ua, ub;
  if (single) {  // a single-point leaf is always direct: its record holds the point itself
    ua = scaled_q(a, u);
    ub = mk4<R>(v.x, v.y, v.z);
  } else {
    const double inv = 1.0 / cnt;
    // centroid = position_sum * (1 / count) (octree.hpp:35)
    ua = scaled_q(a, mk4<R>(R(__dmul_rn(s.a[0], inv)), R(__dmul_rn(s.a[1], inv)),
                            R(__dmul_rn(s.a[2], inv))));
    ub = mk4<R>(R(s.b[0]), R(s.b[1]), R(s.b[2]));
    const V4<R> l = mk4<R>(x.l[0], x.l[1], x.l[2]), h = mk4<R>(x.h[0], x.h[1], x.h[2]);
    if (a.full) {
      st4(a.lo + i, l);
      st4(a.hi + i, h);
      a.s0[i] = make_double4(s.a[0], s.a[1], s.a[2], 0.0);
      a.s1[i] = make_double4(s.b[0], s.b[1], s.b[2], 0.0);
    }
    st4(a.nrec + 4 * i + 2, mk4<R>(l.x, l.y, l.z, ival(R(0), cnt)));
    st4(a.nrec + 4 * i + 3, h);
  }
  ua.w = ival(R(0), code);
  ub.w = ival(R(0), mi.y);
  st4(a.nrec + 4 * i, ua);
  st4(a.nrec + 4 * i + 1, ub);
}

// sum over chunk-local positions [b0, b1] of the staged points, by a warp
// (lane-strided + a fixed butterfly; every lane gets the result)
template <typename R>
__device__ __forceinline__ void warp_range(const V4<R>* su, const V4<R>* sv, int b0, int b1, int lane,
                                           bool box, Sums& s, Box<R>& x) {
  s = Sums{};
  box_init(x);
  for (int t = b0 + lane; t <= b1; t += 32) add_point(s, x, su[t], sv[t], box);
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      s.a[c] += __shfl_xor_sync(0xffffffffu, s.a[c], o);
      s.b[c] += __shfl_xor_sync(0xffffffffu, s.b[c], o);
      x.l[c] = min(x.l[c], __shfl_xor_sync(0xffffffffu, x.l[c], o));
      x.h[c] = max(x.h[c], __shfl_xor_sync(0xffffffffu, x.h[c], o));
    }
}

template <int C>
__device__ __forceinline__ bool is_outer(const int4& mi) {
  return mi.y / C != mi.z / C;
}

// work items of a chunk's warps: a big inside node, the chunk total, a head
// or a tail range
enum { kItemNode = 0, kItemTotal = 1, kItemHead = 2, kItemTail = 3 };

// item slots: [0, kFixItems) heads (<= 33), the total and tails (<= 33);
// [kFixItems, +C/4) big inside nodes -- more than that (chunks of many tight
// clusters, each a chain of nested > 16-point nodes) are summed by their thread
constexpr int kFixItems = 2 * kLevels + 2;
constexpr int kBigSpan = 128;  // chunks: outer nodes spanning more get a CTA in k_agg_outer

template <typename R, int MODE, int C>
__global__ void __launch_bounds__(kNT) k_agg_chunk(const AggArgs<R> a) {
  GS_PDL_ENTRY();
  __shared__ V4<R> su[C], sv[C];
  __shared__ int sl[C + 1];        // sl[1 + j] = lcp(c0 + j, c0 + j + 1); sl[0] = lcp(c0 - 1, c0)
  __shared__ int pm[C];            // pm[j] = min(sl[1 .. 1 + j]) (prefix minimum)
  __shared__ int4 items[kFixItems + C / 4];  // {kind, node / level, b0, b1}
  __shared__ int nitems, nbig;
  const int chunk = blockIdx.x;
  const int64_t c0 = (int64_t)chunk * C;
  const int cl = (int)min((int64_t)C, a.n - c0);
  const int nb = a.first[c0], ne = a.first[c0 + cl];
  // this thread's first node (the usual case: ~1.5 nodes per position),
  // loaded alongside the gather
  const int d0 = nb + (int)threadIdx.x;
  int4 md0 = make_int4(0, 0, 0, 0);
  int nch0 = 0;
  if (d0 < ne) {
    md0 = a.meta[d0];
    nch0 = a.nchild[d0];
  }
  if (threadIdx.x == 0) nitems = nbig = 0;
  // gather the chunk (leaf-order copies on the way): all of this thread's
  // perm loads, then all its record loads, in flight together
  constexpr int kPer = C / kNT;
  int pis[kPer];
#pragma unroll
  for (int r = 0; r < kPer; ++r) {
    const int k = threadIdx.x + r * kNT;
    pis[r] = k < cl ? a.perm[c0 + k] : 0;
  }
  V4<R> us[kPer], vs[kPer];
#pragma unroll
  for (int r = 0; r < kPer; ++r) {
    us[r] = ld4(a.rec + 2 * pis[r]);
    vs[r] = ld4(a.rec + 2 * pis[r] + 1);
  }
#pragma unroll
  for (int r = 0; r < kPer; ++r) {
    const int k = threadIdx.x + r * kNT;
    if (k >= cl) break;
    const int64_t t = c0 + k;
    const V4<R> u = us[r], v = vs[r];
    if (MODE == 0) {
      st4(a.squ + t, mk4<R>(u.x, u.y, u.z));
      st4(a.srec + 2 * t, scaled_q(a, u));
      st4(a.srec + 2 * t + 1, mk4<R>(v.x, v.y, v.z));
    } else {
      st4(a.sadj + 2 * t, u);
      st4(a.sadj + 2 * t + 1, v);
    }
    su[k] = u;
    sv[k] = v;
  }
  for (int k = threadIdx.x; k <= cl; k += kNT) {
    const int64_t t = c0 + k - 1;  // lcp(t, t + 1); none before the first / after the last point
    sl[k] = (t >= 0 && t + 1 < a.n) ? a.lcp[t] : -1;
  }
  __syncthreads();
  // heads: for every level l <= lcp(c0 - 1, c0) the level-l node holding the
  // chunk's first point started earlier; it ends at the first chunk position
  // j with lcp(j, j + 1) < l (a head [0, j]) or covers the whole chunk.
  // j = first position with pm[j] < l: a prefix minimum + binary search.
  const int H = min(sl[0], 32);
  if (H >= 0) {  // (block-uniform)
    for (int k = threadIdx.x; k < C; k += kNT) pm[k] = k < cl ? sl[1 + k] : -1;
    __syncthreads();
    for (int o = 1; o < C; o <<= 1) {  // Hillis-Steele inclusive min-scan
      int v[C / kNT];
#pragma unroll
      for (int r = 0; r < C / kNT; ++r) {
        const int k = threadIdx.x + r * kNT;
        v[r] = k >= o ? min(pm[k], pm[k - o]) : pm[k];
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < C / kNT; ++r) pm[threadIdx.x + r * kNT] = v[r];
      __syncthreads();
    }
    for (int l = threadIdx.x; l <= H; l += kNT) {
      if (pm[cl - 1] >= l) continue;  // covers the whole chunk
      int lo = 0, hi = cl - 1;         // pm non-increasing: first j with pm[j] < l
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (pm[mid] < l) hi = mid;
        else lo = mid + 1;
      }
      items[atomicAdd(&nitems, 1)] = make_int4(kItemHead, l, 0, lo);
    }
  }
  if (threadIdx.x == 0) items[atomicAdd(&nitems, 1)] = make_int4(kItemTotal, 0, 0, cl - 1);
  // the nodes starting in the chunk (the next node's meta loaded one
  // iteration ahead, before this one's work)
  int4 md_cur = md0;
  int nch_cur = nch0;
  for (int d = d0; d < ne; d += kNT) {
    const int4 md = md_cur;
    const int nch = nch_cur;
    if (d + kNT < ne) {
      md_cur = a.meta[d + kNT];
      nch_cur = a.nchild[d + kNT];
    }
    if (is_outer<C>(md)) {  // its tail here; completed by k_agg_outer
      items[atomicAdd(&nitems, 1)] = make_int4(kItemTail, md.w >> 8, md.y - (int)c0, cl - 1);
      if (md.z / C - md.y / C + 1 > kBigSpan) a.outer_big[atomicAdd(a.outer_cnt + 1, 1)] = d;
      else a.outer[atomicAdd(a.outer_cnt, 1)] = d;
      continue;
    }
    const int b0 = md.y - (int)c0, b1 = md.z - (int)c0;
    if (b1 - b0 + 1 > kSmallNode) {
      const int k = atomicAdd(&nbig, 1);
      if (k < C / 4) {
        items[kFixItems + k] = make_int4(kItemNode, d, b0, b1);
        continue;
      }
    }
    Sums s{};
    Box<R> x;
    box_init(x);
    if (!is_single(md))
      for (int t = b0; t <= b1; ++t) add_point(s, x, su[t], sv[t], MODE == 0);
    write_node<R, MODE>(a, d, md, nch, s, x, su[b0], sv[b0]);
  }
  __syncthreads();
  // the warps' items: big inside nodes, the total, heads and tails
  const int lane = threadIdx.x & 31;
  const int nfix = nitems, nall = nfix + min(nbig, C / 4);
  for (int k = threadIdx.x >> 5; k < nall; k += kNT / 32) {
    const int4 it = items[k < nfix ? k : kFixItems + (k - nfix)];
    Sums s;
    Box<R> x;
    warp_range(su, sv, it.z, it.w, lane, MODE == 0, s, x);
    if (lane) continue;
    if (it.x == kItemNode) {
      const int d = it.y;
      write_node<R, MODE>(a, d, a.meta[d], a.nchild[d], s, x, su[it.z], sv[it.z]);
    } else {
      const size_t slot = (size_t)chunk * kPartPerChunk +
                          (it.x == kItemTotal ? 0 : (it.x == kItemHead ? 1 : 1 + kLevels) + it.y);
      a.ps0[slot] = make_double4(s.a[0], s.a[1], s.a[2], 0.0);
      a.ps1[slot] = make_double4(s.b[0], s.b[1], s.b[2], 0.0);
      if (MODE == 0) {
        st4(a.plo + slot, mk4<R>(x.l[0], x.l[1], x.l[2]));
        st4(a.phi + slot, mk4<R>(x.h[0], x.h[1], x.h[2]));
      }
    }
  }
}

// Outer nodes: tail (first chunk) + whole chunks + head (last chunk). One
// warp per node: lanes take the chunk partials strided, a fixed butterfly
// combines them (a fixed order: deterministic).
template <typename R, int MODE, int C>
__global__ void __launch_bounds__(kNT) k_agg_outer(const AggArgs<R> a) {
  GS_PDL_ENTRY();
  const int c = a.outer_cnt[0], cbig = a.outer_cnt[1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const V4<R> z = mk4<R>(0, 0, 0);
  // nodes spanning many chunks (the root spans all): a CTA each, chunks
  // strided over its threads, then warp butterflies and the 8 warp sums in
  // order (fixed: deterministic)
  for (int k = blockIdx.x; k < cbig; k += gridDim.x) {
    const int d = a.outer_big[k];
    const int4 md = a.meta[d];
    const int lev = md.w >> 8, cb = md.y / C, ce = md.z / C;
    Sums s{};
    Box<R> x;
    box_init(x);
#pragma unroll 2
    for (int ch = cb + (int)threadIdx.x; ch <= ce; ch += kNT) {
      const size_t slot = (size_t)ch * kPartPerChunk +
                          (ch == cb ? 1 + kLevels + lev : (ch == ce ? 1 + lev : 0));
      add_part(s, x, ldcg4(a.ps0 + slot), ldcg4(a.ps1 + slot),
               MODE == 0 ? ldcg4(a.plo + slot) : z, MODE == 0 ? ldcg4(a.phi + slot) : z);
    }
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        s.a[q] += __shfl_xor_sync(0xffffffffu, s.a[q], o);
        s.b[q] += __shfl_xor_sync(0xffffffffu, s.b[q], o);
        x.l[q] = min(x.l[q], __shfl_xor_sync(0xffffffffu, x.l[q], o));
        x.h[q] = max(x.h[q], __shfl_xor_sync(0xffffffffu, x.h[q], o));
      }
    __shared__ double ws[kNT / 32][6];
    __shared__ R wb[kNT / 32][6];
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        ws[warp][q] = s.a[q];
        ws[warp][3 + q] = s.b[q];
        wb[warp][q] = x.l[q];
        wb[warp][3 + q] = x.h[q];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      Sums t{};
      Box<R> y;
      box_init(y);
      for (int w = 0; w < kNT / 32; ++w)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          t.a[q] += ws[w][q];
          t.b[q] += ws[w][3 + q];
          y.l[q] = min(y.l[q], wb[w][q]);
          y.h[q] = max(y.h[q], wb[w][3 + q]);
        }
      write_node<R, MODE>(a, d, md, a.nchild[d], t, y, z, z);
    }
    __syncthreads();
  }
  for (int k = (blockIdx.x * kNT + threadIdx.x) >> 5; k < c; k += (gridDim.x * kNT) >> 5) {
    const int d = a.outer[k];
    const int4 md = a.meta[d];
    const int lev = md.w >> 8, cb = md.y / C, ce = md.z / C;
    Sums s{};
    Box<R> x;
    box_init(x);
    // slot sequence: tail(cb), total(cb + 1 .. ce - 1), head(ce)
#pragma unroll 2
    for (int ch = cb + lane; ch <= ce; ch += 32) {
      const size_t slot = (size_t)ch * kPartPerChunk +
                          (ch == cb ? 1 + kLevels + lev : (ch == ce ? 1 + lev : 0));
      add_part(s, x, ldcg4(a.ps0 + slot), ldcg4(a.ps1 + slot),
               MODE == 0 ? ldcg4(a.plo + slot) : z, MODE == 0 ? ldcg4(a.phi + slot) : z);
    }
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        s.a[q] += __shfl_xor_sync(0xffffffffu, s.a[q], o);
        s.b[q] += __shfl_xor_sync(0xffffffffu, s.b[q], o);
        x.l[q] = min(x.l[q], __shfl_xor_sync(0xffffffffu, x.l[q], o));
        x.h[q] = max(x.h[q], __shfl_xor_sync(0xffffffffu, x.h[q], o));
      }
    if (lane == 0) write_node<R, MODE>(a, d, md, a.nchild[d], s, x, z, z);
  }
}

// traversal-format node fields: centroid = position_sum * (1 / count)
// (octree.hpp:35), scaled for FP32; momentum sum; adjoint sum / beta mean.
// Traversal record (4 vec4 per node):
//   {centroid | point, code} {momentum sum | p, begin} {lo.xyz, count} {hi.xyz, -},
//   code = skip | single-point leaf << 31 | bucket leaf << 30 | twig << 29
//   (skip < 2^29: tree_build caps n accordingly): 64 B (FP32), loaded whole
//   by two 256-bit loads; the first half is the node's interaction unit.
template <typename R>
__global__ void k_finalize(int mode, const int4* meta, const int* mp, const double4* s0,
                           const double4* s1, double kap, double c0x, double c0y, double c0z,
                           int scaled, V4<R>* o0, V4<R>* o1, const V4<R>* lo = nullptr,
                           const V4<R>* hi = nullptr, V4<R>* nrec = nullptr,
                           const V4<R>* srec = nullptr, const int* nchild = nullptr) {
  const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
  if (i >= *mp) return;
  const int4 mi = meta[i];
  const int cnt = mi.z - mi.y + 1;
  const double inv = 1.0 / cnt;
  const bool single = (mi.w & 1) && cnt == 1;  // no stored sums (k_aggregate)
  const double4 z4 = make_double4(0, 0, 0, 0);
  const double4 a = single ? z4 : s0[i], b = single ? z4 : s1[i];
  if (mode == 0) {
    double cx = __dmul_rn(a.x, inv), cy = __dmul_rn(a.y, inv), cz = __dmul_rn(a.z, inv);
    const V4<R> cen = scaled ? mk4<R>((R)fmaf((float)kap, (float)cx, -(float)(kap * c0x)),
                                      (R)fmaf((float)kap, (float)cy, -(float)(kap * c0y)),
                                      (R)fmaf((float)kap, (float)cz, -(float)(kap * c0z)), R(cnt))
                             : mk4<R>(R(cx), R(cy), R(cz), R(cnt));
    const V4<R> mom = mk4<R>(R(b.x), R(b.y), R(b.z), ival(R(0), cnt));
    if (nrec) {
      const bool leaf = mi.w & 1;
      // twig: an internal node whose children are all leaves (subtree = itself +
      // its children); opening it makes every point of it direct, no child gated
      const bool twig = !leaf && nchild && nchild[i] == 0;
      const int code = mi.x | (single ? (int)0x80000000u : 0) | ((leaf && cnt > 1) ? 0x40000000 : 0) |
                       (twig ? 0x20000000 : 0);
      // half A = the unit this node contributes: its centroid and momentum sum,
      // or -- a single-point leaf being always direct (leaf-first,
      // bh_kernel.cpp:40-45) -- the point itself; the walk loads it straight
      // into the interaction operands. Half B = the tight box for the gate.
      V4<R> ua = single ? ld4(srec + 2 * mi.y) : cen;
      V4<R> ub = single ? ld4(srec + 2 * mi.y + 1) : mom;
      ua.w = ival(R(0), code);
      ub.w = ival(R(0), mi.y);
      st4(nrec + 4 * i, ua);
      st4(nrec + 4 * i + 1, ub);
      if (!single) {
        V4<R> l = ld4(lo + i);
        l.w = ival(R(0), cnt);
        st4(nrec + 4 * i + 2, l);
        st4(nrec + 4 * i + 3, ld4(hi + i));
      }
    }
  } else {
    // interleaved {alpha sum, beta mean} per node (one 256-bit load in the walk);
    // for a single-point leaf these are exactly the point's alpha and beta
    // (read from the leaf-order adjoints, passed as srec)
    if (single) {
      st4(o0 + 2 * i, ld4(srec + 2 * mi.y));
      st4(o0 + 2 * i + 1, ld4(srec + 2 * mi.y + 1));
      return;
    }
    st4(o0 + 2 * i, mk4<R>(R(a.x), R(a.y), R(a.z)));
    // db = beta_i - (1 / count) * beta_sum, bh_kernel.cpp:146
    st4(o0 + 2 * i + 1, mk4<R>(R(__dmul_rn(inv, b.x)), R(__dmul_rn(inv, b.y)), R(__dmul_rn(inv, b.z))));
    (void)o1;
  }
}

// cell box of a node: replay its key prefix from the root box
__global__ void k_cells(const int4* meta, int64_t m, const uint64_t* skh, const uint64_t* skl,
                        const double* root, double* boxes) {
  const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
  if (i >= m) return;
  const int4 mi = meta[i];
  const int level = mi.w >> 8;
  const uint64_t h = skh[mi.y], l = skl[mi.y];
  double lo[3] = {root[0], root[1], root[2]}, hi[3] = {root[3], root[4], root[5]};
  for (int lev = 1; lev <= level; ++lev) {
    const unsigned dig = lev <= 21 ? (unsigned)(h >> (3 * (21 - lev))) & 7u
                                   : (unsigned)(l >> (3 * (32 - lev))) & 7u;
    for (int a = 0; a < 3; ++a) {
      const double c = __dmul_rn(0.5, __dadd_rn(lo[a], hi[a]));
      if ((dig >> a) & 1u) lo[a] = c;
      else hi[a] = c;
    }
  }
  for (int a = 0; a < 3; ++a) {
    boxes[12 * i + a] = lo[a];
    boxes[12 * i + 3 + a] = hi[a];
  }
}

// first[0..n]: exclusive scan of the node counts per position (computed
// inline from the lcp array; first[n] = node count). One pass: 1024-position
// tiles (4096 positions) in the order of an atomic ticket, each publishing its sum and then
// its inclusive prefix (flag << 30 | value), a warp looking back over 32
// predecessors per round trip.
constexpr unsigned kScanAgg = 1u << 30, kScanPre = 2u << 30, kScanVal = (1u << 30) - 1;
constexpr int kScanIPT = 4;  // positions per thread: 4096-position tiles
__global__ void __launch_bounds__(1024) k_scan_nodes(const int* L, int64_t n, int* out,
                                                     unsigned* desc, unsigned* ticket) {
  GS_PDL_ENTRY();
  __shared__ int s_tile;
  __shared__ int ws[32];
  __shared__ unsigned s_excl;
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(ticket, 1u);
  __syncthreads();
  const int tile = s_tile;
  const int64_t i0 = (tile * 1024LL + threadIdx.x) * kScanIPT;  // this thread's positions
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int cnt[kScanIPT], v = 0;
#pragma unroll
  for (int k = 0; k < kScanIPT; ++k) {
    cnt[k] = 0;
    if (i0 + k < n) {
      int Lm, Lp, ci, lf;
      starts(L, n, i0 + k, Lm, Lp, ci, lf);
      cnt[k] = ci + lf;
    }
    v += cnt[k];
  }
  int x = v;  // inclusive block scan of the per-thread sums
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += u;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = ws[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += u;
    }
    ws[lane] = w;  // inclusive over warps
    const unsigned total = (unsigned)__shfl_sync(0xffffffffu, w, 31);
    cuda::atomic_ref<unsigned, cuda::thread_scope_device> mine(desc[tile]);
    unsigned excl = 0;
    if (tile == 0) {
      if (lane == 0) mine.store(kScanPre | total, cuda::memory_order_release);
    } else {
      if (lane == 0) mine.store(kScanAgg | total, cuda::memory_order_release);
      for (int t = tile - 1; t >= 0;) {
        const int p = t - lane;
        unsigned st = kScanPre;  // (before tile 0: never consulted)
        if (p >= 0) {
          cuda::atomic_ref<unsigned, cuda::thread_scope_device> d(desc[p]);
          st = d.load(cuda::memory_order_acquire);
        }
        const unsigned ready = __ballot_sync(0xffffffffu, (st & (kScanAgg | kScanPre)) != 0);
        const unsigned pre = __ballot_sync(0xffffffffu, (st & kScanPre) != 0);
        // lanes up to the nearest prefix must all have published
        const int stop = pre ? __ffs(pre) - 1 : 31;
        const unsigned need = stop == 31 ? 0xffffffffu : ((2u << stop) - 1u);
        if ((ready & need) != need) continue;  // poll the same window again
        unsigned add = lane <= stop ? (st & kScanVal) : 0u;
        for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
        excl += add;
        if (pre) break;
        t -= 32;
      }
      if (lane == 0) mine.store(kScanPre | (excl + total), cuda::memory_order_release);
    }
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  int run = (int)s_excl + (warp ? ws[warp - 1] : 0) + x - v;
#pragma unroll
  for (int k = 0; k < kScanIPT; ++k) {
    if (i0 + k < n) out[i0 + k] = run;
    run += cnt[k];
    if (i0 + k == n - 1) out[n] = run;
  }
}

}  // namespace

int tree_finalize_fwd(int prec, DevTree& t, const KernelConsts& kc, cudaStream_t st);

// Node aggregates + traversal records: mode 0 (boxes, sums of q and p, nrec;
// the leaf-order copies srec / squ of the records `src`), mode 1 (sums of
// alpha and beta, nadj; the leaf-order copy sadj of the adjoints `src`).
// chunk of C leaf-order points per CTA: 256 below 256k points (more CTAs in
// flight), else 1024 (FP32) / 512 (FP64)
template <typename R, int C>
static int aggregate_t(int mode, DevTree& t, const void* src, const KernelConsts& kc, cudaStream_t st) {
  const int64_t nch = (t.n + C - 1) / C;
  AggArgs<R> a{};
  a.meta = t.meta.as<int4>();
  a.nchild = t.nchild.as<int>();
  a.first = t.first.as<int>();
  a.lcp = t.lcp.as<int>();
  a.perm = t.perm.as<int>();
  a.n = t.n;
  a.rec = static_cast<const V4<R>*>(src);
  a.kap = kc.kappa;
  a.c0x = kc.c0[0];
  a.c0y = kc.c0[1];
  a.c0z = kc.c0[2];
  a.scaled = sizeof(R) == 4;
  a.full = !t.lean;
  const size_t parts = (size_t)nch * kPartPerChunk;
  GS_TRY_INT(t.parts.ensure(parts * (2 * sizeof(double4) + 2 * sizeof(V4<R>))));
  a.ps0 = t.parts.as<double4>();
  a.ps1 = a.ps0 + parts;
  a.plo = reinterpret_cast<V4<R>*>(a.ps1 + parts);
  a.phi = a.plo + parts;
  // outer nodes: per level at most one starts in each chunk
  // (per level at most one outer node starts in a chunk; those spanning more
  // than kBigSpan chunks are at most one per kBigSpan chunks per level)
  const size_t nbig_cap = (size_t)kLevels * (nch / kBigSpan + 2);
  GS_TRY_INT(t.outer.ensure(sizeof(int) * (64 + kLevels * (nch + 1) + nbig_cap)));
  a.outer_cnt = t.outer.as<int>();
  a.outer = a.outer_cnt + 64;
  a.outer_big = a.outer + kLevels * (nch + 1);
  GS_CUDA_OK(cudaMemsetAsync(a.outer_cnt, 0, 2 * sizeof(int), st));
  if (mode == 0) {
    a.srec = t.srec.as<V4<R>>();
    a.squ = t.squ.as<V4<R>>();
    a.lo = t.lo.as<V4<R>>();
    a.hi = t.hi.as<V4<R>>();
    a.s0 = t.psum.as<double4>();
    a.s1 = t.msum.as<double4>();
    a.nrec = t.nrec.as<V4<R>>();
    GS_CUDA_OK(pdl_launch(k_agg_chunk<R, 0, C>, (unsigned)nch, kNT, 0, st, a));
    GS_CUDA_OK(pdl_launch(k_agg_outer<R, 0, C>, 4 * 148, kNT, 0, st, a));
  } else {
    a.sadj = t.sadj.as<V4<R>>();
    a.s0 = t.asum.as<double4>();
    a.s1 = t.bsum.as<double4>();
    a.nadj = t.nadj.as<V4<R>>();
    GS_CUDA_OK(pdl_launch(k_agg_chunk<R, 1, C>, (unsigned)nch, kNT, 0, st, a));
    GS_CUDA_OK(pdl_launch(k_agg_outer<R, 1, C>, 4 * 148, kNT, 0, st, a));
  }
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}

static int aggregate(int mode, int prec, DevTree& t, const void* src, const KernelConsts& kc,
                     cudaStream_t st) {
  static const int forced = [] {  // GS_AGG_CHUNK: 256 / 512 / 1024 (experiments)
    const char* e = std::getenv("GS_AGG_CHUNK");
    return e ? std::atoi(e) : 0;
  }();
  const int C = forced ? forced : (t.n <= (1 << 18) ? 256 : (prec == kF32 ? 1024 : 512));
  if (prec == kF32) {
    if (C == 256) return aggregate_t<float, 256>(mode, t, src, kc, st);
    if (C == 512) return aggregate_t<float, 512>(mode, t, src, kc, st);
    return aggregate_t<float, 1024>(mode, t, src, kc, st);
  }
  if (C == 256) return aggregate_t<double, 256>(mode, t, src, kc, st);
  return aggregate_t<double, 512>(mode, t, src, kc, st);
}

// first[0..n] (out[n] = m) by k_scan_nodes; desc / ticket: zeroed scratch
static int scan_ints(const int* L, int64_t n, int* out, unsigned* desc, unsigned* ticket,
                     cudaStream_t st) {
  GS_CUDA_OK(pdl_launch(k_scan_nodes, nblocks(n, 1024 * kScanIPT), 1024, 0, st, L, n, out, desc, ticket));
  return GS_OK;
}

// k_tie_sort as a cooperative launch: as many CTAs as can be co-resident (at
// most 2 per SM), so grid.sync() is legal
static int tie_sort(const Device& dev, DevTree& t, const void* rec, unsigned* ctr, cudaStream_t st) {
  static int per_sm = 0;
  void* fn = (void*)k_tie_sort;
  if (!per_sm) {
    int b = 0;
    GS_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kNT, 0));
    per_sm = std::max(1, std::min(2, b));
  }
  const int grid = std::max(1, std::min(nblocks(t.n, kNT), per_sm * dev.sms));
  TieKeys klo{t.key_lo.as<uint64_t>(), rec, t.root.as<double>(), t.skey_hi.as<uint64_t>(),
              t.prec == kF32 ? 1 : 0, 1};
  const unsigned* lo_valid = t.klo_flag.as<unsigned>();
  const int2* small_runs = (const int2*)t.tmp_v.ptr;
  int4* big_runs = (int4*)t.tmp_v2.ptr;
  int* perm = t.perm.as<int>();
  uint64_t* skl = t.skey_lo.as<uint64_t>();
  uint64_t* bufa = t.tmp_k.as<uint64_t>();
  GS_TRY_INT(t.tie_buf.ensure(8 * (size_t)t.n));
  uint64_t* bufb = t.tie_buf.as<uint64_t>();
  // scratch of the long-run radix passes: slots (chunks of runs > 2048 points,
  // <= n / 1024, each run padded to whole groups of kTieGroup: <= 8.5 n / 1024)
  // x 256 digit counts + 2 x groups x 256 group sums: < 2.5 n words
  GS_TRY_INT(t.tie_scr.ensure(sizeof(unsigned) * (3 * (size_t)t.n + 4096)));
  unsigned* chist = t.tie_scr.as<unsigned>();
  const unsigned* cctr = ctr;
  int* L = t.lcp.as<int>();
  void* args[] = {(void*)&klo, (void*)&lo_valid, (void*)&cctr, (void*)&small_runs, (void*)&big_runs,
                  (void*)&perm, (void*)&skl, (void*)&bufa, (void*)&bufb, (void*)&chist, (void*)&L};
  GS_CUDA_OK(cudaLaunchCooperativeKernel(fn, grid, kNT, args, 0, st));
  return GS_OK;
}

int tree_build(const Device& dev, int prec, const KernelConsts& kc, const void* rec, int64_t n,
               DevTree& t, cudaStream_t st, const double* root_box, int* overflow) {
  t.prec = prec;
  t.n = n;
  t.kc = kc;
  t.adj_valid = false;
  const size_t vb = vec_bytes(prec);
  GS_TRY_INT(t.key_hi.ensure(8 * n));
  GS_TRY_INT(t.key_lo.ensure(8 * n));
  GS_TRY_INT(t.perm.ensure(4 * n));
  GS_TRY_INT(t.skey_hi.ensure(8 * n));
  GS_TRY_INT(t.skey_lo.ensure(8 * n));
  GS_TRY_INT(t.lcp.ensure(4 * (n + 1)));
  GS_TRY_INT(t.first.ensure(4 * (n + 2)));
  GS_TRY_INT(t.srec.ensure(2 * vb * n));
  GS_TRY_INT(t.tmp_k.ensure(8 * n));
  GS_TRY_INT(t.tmp_v.ensure(4 * n));
  GS_TRY_INT(t.root.ensure(8 * 8));
  GS_TRY_INT(t.scal.ensure(64));
  const int bb = std::min(nblocks(n, kNT), 2 * dev.sms);
  GS_TRY_INT(t.scan_tmp.ensure(sizeof(double) * 6 * bb + 64));
  {  // k_bbox's arrival counter: zeroed when allocated, then reset by each last block
    void* before = t.bbox_ctr.ptr;
    GS_TRY_INT(t.bbox_ctr.ensure(16));
    if (t.bbox_ctr.ptr != before) GS_CUDA_OK(cudaMemsetAsync(t.bbox_ctr.ptr, 0, 16, st));
  }
  kt_mark(2, st);
  // 1. padded root box (or the caller's explicit root cell)
  if (root_box) {
    GS_CUDA_OK(cudaMemcpyAsync(t.root.ptr, root_box, 6 * sizeof(double), cudaMemcpyHostToDevice, st));
  } else {
    if (prec == kF32) GS_CUDA_OK(pdl_launch(k_bbox<float>, bb, kNT, 0, st, (const float4*)rec, n, t.scan_tmp.as<double>(), t.bbox_ctr.as<unsigned>(), t.root.as<double>()));
    else GS_CUDA_OK(pdl_launch(k_bbox<double>, bb, kNT, 0, st, (const double4*)rec, n, t.scan_tmp.as<double>(), t.bbox_ctr.as<unsigned>(), t.root.as<double>()));
  }
  // 2. keys (the deep key too when the previous build of this tree had ties:
  // its tie flag is still in the sort scratch, whose counters sit at a fixed
  // offset; no scratch yet -> compute it)
  const int nb = nblocks(n, kNT);
  GS_TRY_INT(t.klo_flag.ensure(16));
  static const int keys_lo_env = [] {  // GS_KEYS_LO: 0 never (tests the tie sort's replay), 1 always
    const char* e = std::getenv("GS_KEYS_LO");
    return e ? std::atoi(e) : -1;
  }();
  GS_TRY_INT(t.scal.ensure(64));
  if (keys_lo_env >= 0) {  // a constant "previous tie flag" (scal word 8; static source:
                           // a captured copy replays from it)
    static const unsigned v = (unsigned)keys_lo_env;
    GS_CUDA_OK(cudaMemcpyAsync(t.scal.as<unsigned>() + 8, &v, sizeof v, cudaMemcpyHostToDevice, st));
  }
  const unsigned* want_lo = keys_lo_env >= 0 ? t.scal.as<unsigned>() + 8
                            : (t.hist.ptr ? t.hist.as<unsigned>() + kHistWords + kTieFlag : nullptr);
  if (prec == kF32)
    GS_CUDA_OK(pdl_launch(k_keys<float>, nb, kNT, 0, st, (const float4*)rec, n, t.root.as<double>(), t.key_hi.as<uint64_t>(), t.key_lo.as<uint64_t>(), want_lo, t.klo_flag.as<unsigned>()));
  else
    GS_CUDA_OK(pdl_launch(k_keys<double>, nb, kNT, 0, st, (const double4*)rec, n, t.root.as<double>(), t.key_hi.as<uint64_t>(), t.key_lo.as<uint64_t>(), want_lo, t.klo_flag.as<unsigned>()));
  GS_CUDA_OK(cudaGetLastError());
  kt_mark(2, st);
  kt_mark(3, st);
  // 3. order by the full key (key_hi, key_lo, index): a stable LSD radix sort
  // of key_hi with the index as value -- 8 passes of 8-bit digits, ping-pong
  //   (key_hi, index) -> (tmp_k, tmp_v2) -> (skey_hi, perm) -> ... -> (skey_hi, perm)
  // -- then the runs of equal key_hi (only below the 21st level: duplicates,
  // depth-32 clusters) sorted in place by (key_lo, index) (k_tie_runs/_sort).
  // keys per thread: small tiles (more CTAs) for small n, 8 from ~0.5M points
  static const int ipt_env = [] {
    const char* e = std::getenv("GS_RS_IPT");
    const int v = e ? std::atoi(e) : 0;
    return (v == 4 || v == 8) ? v : 0;
  }();
  static const int nt_env = [] {  // GS_RS_NT: 256 / 512 threads per one-sweep tile
    const char* e = std::getenv("GS_RS_NT");
    const int v = e ? std::atoi(e) : 0;
    return (v == 256 || v == 512 || v == 1024) ? v : 0;
  }();
  const int ipt = ipt_env ? ipt_env : (n >= (1 << 19) ? 8 : 4);
  // the biggest tiles that still fit one wave -- 1024 x 8 (one per SM) up to
  // ~1.2M points, else 512 x 8 (two per SM), else 256 x 8: fewer tiles, a
  // shorter look-back chain (1M: sort 0.197 -> 0.176 -> 0.169 ms for 489 ->
  // 245 -> 123 tiles); beyond one wave of any, 256 x 8 (4M: 0.54 vs 0.56 ms)
  int auto_nt = 256;
  if (ipt == 8 && nblocks(n, 1024 * ipt) <= dev.sms) auto_nt = 1024;
  else if (ipt == 8 && nblocks(n, 512 * ipt) <= 2 * dev.sms) auto_nt = 512;
  const int rs_nt = nt_env ? (nt_env > 256 && ipt == 8 ? nt_env : 256) : auto_nt;
  const int ntiles = nblocks(n, rs_nt * ipt);
  const int hblocks = nblocks(n, kRsNT * ipt);  // k_rs_hist_all: 256 x IPT keys per block
  GS_TRY_INT(t.tmp_v2.ensure(4 * n));
  // digits: 9 bits (7 passes over the 63-bit key) with the 1024-thread tiles
  // (one digit per thread; 1M: sort 0.168 -> 0.162 ms), else 8 bits (8 passes)
  static const int bits_env = [] {
    const char* e = std::getenv("GS_RS_BITS");
    const int v = e ? std::atoi(e) : 0;
    return (v == 8 || v == 9) ? v : 0;
  }();
  const int bits = rs_nt == 1024 ? (bits_env ? bits_env : 9) : 8;
  const int npass = (63 + bits - 1) / bits, dig = 1 << bits;
  // one-sweep scratch: the passes' digit histograms (kHistWords), 32 counters
  // (the passes' tile counters; the tie lists' counters and flag -- a fixed
  // offset, read by the next build's k_keys), npass x ntiles x dig look-back
  // status words, the node scan's look-back words -- zeroed by one memset
  const size_t words = (size_t)kHistWords + 32 + (size_t)npass * ntiles * dig + nblocks(n, 1024);
  GS_TRY_INT(t.hist.ensure(sizeof(unsigned) * words));
  GS_CUDA_OK(cudaMemsetAsync(t.hist.ptr, 0, sizeof(unsigned) * words, st));
  unsigned* hist = t.hist.as<unsigned>();
  unsigned* ctr = hist + kHistWords;
  unsigned* desc = ctr + 32;
  if (bits == 9) GS_CUDA_OK(pdl_launch(k_rs_hist_all<8, 9>, hblocks, kRsNT, 0, st, t.key_hi.as<uint64_t>(), n, hist));
  else if (ipt == 8) GS_CUDA_OK(pdl_launch(k_rs_hist_all<8>, hblocks, kRsNT, 0, st, t.key_hi.as<uint64_t>(), n, hist));
  else GS_CUDA_OK(pdl_launch(k_rs_hist_all<4>, hblocks, kRsNT, 0, st, t.key_hi.as<uint64_t>(), n, hist));
  {
    const uint64_t* ka = t.key_hi.as<uint64_t>();
    const int* va = nullptr;  // first pass: the value is the index
    for (int p = 0; p < npass; ++p) {
      // ping-pong so that the last pass lands in (skey_hi, perm)
      const bool to_final = ((npass - 1 - p) & 1) == 0;
      uint64_t* kb = to_final ? t.skey_hi.as<uint64_t>() : t.tmp_k.as<uint64_t>();
      int* vb = to_final ? t.perm.as<int>() : t.tmp_v2.as<int>();
      GS_TRY_INT(onesweep(ipt, rs_nt, ntiles, st, ka, va, kb, vb, n, bits * p, hist + p * dig,
               desc + (size_t)p * ntiles * dig, ctr + p, bits));
      ka = kb;
      va = vb;
    }
  }
  // ties: runs of equal key_hi sorted by (key_lo, index) in place (perm,
  // skey_lo of the run members); tmp_v / tmp_v2 hold the run lists, tmp_k /
  // key_lo the long runs' merge buffers (all free after the key_hi sort)
  GS_CUDA_OK(pdl_launch(k_lcp_runs, nb, kNT, 0, st, t.skey_hi.as<uint64_t>(), n, t.lcp.as<int>(), ctr,
                        (int2*)t.tmp_v.ptr, (int4*)t.tmp_v2.ptr));
  GS_TRY_INT(tie_sort(dev, t, rec, ctr, st));
  GS_CUDA_OK(cudaGetLastError());
  kt_mark(3, st);
  kt_mark(4, st);
  // 4. topology
  GS_TRY_INT(scan_ints(t.lcp.as<int>(), n, t.first.as<int>(), desc + (size_t)npass * ntiles * dig,
                       ctr + kScanTicket, st));
  // The node count m = first[n] stays on the device: node arrays are sized
  // for 4n + 64 nodes (m ~ 1.5n for volumes and surfaces) and every kernel
  // reads m from first[n]; more nodes than that (degenerate clustering) raise
  // *overflow instead of writing out of bounds. No host round trip per build.
  t.m = -1;
  const int64_t cap = 4 * n + 64;
  if (cap >= (int64_t(1) << 29)) return GS_INVALID_ARGUMENT;  // node index must fit the 29-bit skip field
  t.cap = cap;
  GS_TRY_INT(t.meta.ensure(sizeof(int4) * cap));
  GS_TRY_INT(t.parent.ensure(4 * cap));
  GS_TRY_INT(t.nchild.ensure(4 * cap));
  GS_TRY_INT(t.lo.ensure(vb * cap));
  GS_TRY_INT(t.hi.ensure(vb * cap));
  GS_TRY_INT(t.nrec.ensure(4 * vb * cap));
  GS_TRY_INT(t.psum.ensure(sizeof(double4) * cap));
  GS_TRY_INT(t.msum.ensure(sizeof(double4) * cap));
  GS_TRY_INT(t.squ.ensure(vb * n));
  const int mb = nblocks(cap, kNT);
  GS_TRY_INT(t.start.ensure(4 * cap));
  GS_CUDA_OK(pdl_launch(k_node_starts, nb, kNT, 0, st, t.first.as<int>(), n, cap, t.start.as<int>(),
                        overflow));
  GS_CUDA_OK(pdl_launch(k_nodes, mb, kNT, 0, st, t.skey_hi.as<uint64_t>(), t.skey_lo.as<uint64_t>(), t.lcp.as<int>(),
                              t.first.as<int>(), t.start.as<int>(), n, cap, t.meta.as<int4>(),
                              t.parent.as<int>(), t.nchild.as<int>(), t.lean ? 0 : 1));
  GS_CUDA_OK(cudaGetLastError());
  kt_mark(4, st);
  kt_mark(5, st);
  // 5. leaf-order records + aggregates + traversal records, one kernel
  GS_TRY_INT(aggregate(0, prec, t, rec, kc, st));
  kt_mark(5, st);
  return GS_OK;
}

// Points in Morton (leaf) order for locality only -- the exact path's
// underflow cutoff (allpairs.cu): bbox, 63-bit keys, an 8-pass index-stable
// radix sort on them, then the leaf-order copy of the records (t.srec: FP32
// interaction coordinates, p) and t.perm. No topology, no aggregates.
int morton_order(const Device& dev, int prec, const KernelConsts& kc, const void* rec, int64_t n,
                 DevTree& t, cudaStream_t st) {
  t.prec = prec;
  t.n = n;
  t.kc = kc;
  const size_t vb = vec_bytes(prec);
  GS_TRY_INT(t.key_hi.ensure(8 * n));
  GS_TRY_INT(t.key_lo.ensure(8 * n));
  GS_TRY_INT(t.skey_hi.ensure(8 * n));
  GS_TRY_INT(t.perm.ensure(4 * n));
  GS_TRY_INT(t.tmp_k.ensure(8 * n));
  GS_TRY_INT(t.tmp_v.ensure(4 * n));
  GS_TRY_INT(t.root.ensure(8 * 8));
  GS_TRY_INT(t.srec.ensure(2 * vb * n));
  GS_TRY_INT(t.squ.ensure(vb * n));
  const int bb = std::min(nblocks(n, kNT), 2 * dev.sms);
  GS_TRY_INT(t.scan_tmp.ensure(sizeof(double) * 6 * bb + 64));
  {  // k_bbox's arrival counter: zeroed when allocated, then reset by each last block
    void* before = t.bbox_ctr.ptr;
    GS_TRY_INT(t.bbox_ctr.ensure(16));
    if (t.bbox_ctr.ptr != before) GS_CUDA_OK(cudaMemsetAsync(t.bbox_ctr.ptr, 0, 16, st));
  }
  if (prec == kF32) GS_CUDA_OK(pdl_launch(k_bbox<float>, bb, kNT, 0, st, (const float4*)rec, n, t.scan_tmp.as<double>(), t.bbox_ctr.as<unsigned>(), t.root.as<double>()));
  else GS_CUDA_OK(pdl_launch(k_bbox<double>, bb, kNT, 0, st, (const double4*)rec, n, t.scan_tmp.as<double>(), t.bbox_ctr.as<unsigned>(), t.root.as<double>()));
  const int nb = nblocks(n, kNT);
  GS_TRY_INT(t.klo_flag.ensure(16));
  if (prec == kF32)
    GS_CUDA_OK(pdl_launch(k_keys<float>, nb, kNT, 0, st, (const float4*)rec, n, t.root.as<double>(), t.key_hi.as<uint64_t>(), t.key_lo.as<uint64_t>(), nullptr, t.klo_flag.as<unsigned>()));
  else
    GS_CUDA_OK(pdl_launch(k_keys<double>, nb, kNT, 0, st, (const double4*)rec, n, t.root.as<double>(), t.key_hi.as<uint64_t>(), t.key_lo.as<uint64_t>(), nullptr, t.klo_flag.as<unsigned>()));
  const int ipt = n >= (1 << 19) ? 8 : 4;
  const int ntiles = nblocks(n, kRsNT * ipt);
  const size_t words = (size_t)kHistWords + 32 + (size_t)8 * ntiles * 256;
  GS_TRY_INT(t.hist.ensure(sizeof(unsigned) * words));
  GS_CUDA_OK(cudaMemsetAsync(t.hist.ptr, 0, sizeof(unsigned) * words, st));
  unsigned* hist = t.hist.as<unsigned>();
  unsigned* ctr = hist + kHistWords;
  unsigned* desc = ctr + 32;
  if (ipt == 8) GS_CUDA_OK(pdl_launch(k_rs_hist_all<8>, ntiles, kRsNT, 0, st, t.key_hi.as<uint64_t>(), n, hist));
  else GS_CUDA_OK(pdl_launch(k_rs_hist_all<4>, ntiles, kRsNT, 0, st, t.key_hi.as<uint64_t>(), n, hist));
  const uint64_t* ka = t.key_hi.as<uint64_t>();
  const int* va = nullptr;
  for (int p = 0; p < 8; ++p) {  // (key_hi, index) -> (tmp_k, tmp_v) -> (skey_hi, perm) -> ...
    uint64_t* kb = (p & 1) ? t.skey_hi.as<uint64_t>() : t.tmp_k.as<uint64_t>();
    int* vb2 = (p & 1) ? t.perm.as<int>() : t.tmp_v.as<int>();
    unsigned* dq = desc + (size_t)p * ntiles * 256;
    GS_TRY_INT(onesweep(ipt, 256, ntiles, st, ka, va, kb, vb2, n, 8 * p, hist + p * 256, dq, ctr + p));
    ka = kb;
    va = vb2;
  }
  if (prec == kF32)
    GS_CUDA_OK(pdl_launch(k_gather<float>, nb, kNT, 0, st, (const float4*)rec, t.perm.as<int>(), n, kc.kappa, kc.c0[0], kc.c0[1], kc.c0[2], 1, t.srec.as<float4>(), t.squ.as<float4>()));
  else
    GS_CUDA_OK(pdl_launch(k_gather<double>, nb, kNT, 0, st, (const double4*)rec, t.perm.as<int>(), n, kc.kappa, kc.c0[0], kc.c0[1], kc.c0[2], 0, t.srec.as<double4>(), t.squ.as<double4>()));
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}

int tree_finalize_fwd(int prec, DevTree& t, const KernelConsts& kc, cudaStream_t st) {
  const int* mp = t.first.as<int>() + t.n;
  const int mb = nblocks(t.cap, kNT);
  const int scaled = prec == kF32;
  t.kc = kc;
  if (prec == kF32)
    k_finalize<float><<<mb, kNT, 0, st>>>(0, t.meta.as<int4>(), mp, t.psum.as<double4>(), t.msum.as<double4>(), kc.kappa, kc.c0[0], kc.c0[1], kc.c0[2], scaled, t.cen.as<float4>(), t.mom.as<float4>(), t.lo.as<float4>(), t.hi.as<float4>(), t.nrec.as<float4>(), t.srec.as<float4>(), t.nchild.as<int>());
  else
    k_finalize<double><<<mb, kNT, 0, st>>>(0, t.meta.as<int4>(), mp, t.psum.as<double4>(), t.msum.as<double4>(), kc.kappa, kc.c0[0], kc.c0[1], kc.c0[2], scaled, t.cen.as<double4>(), t.mom.as<double4>(), t.lo.as<double4>(), t.hi.as<double4>(), t.nrec.as<double4>(), t.srec.as<double4>(), t.nchild.as<int>());
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}

int tree_rescale(int prec, DevTree& t, const void* rec, const KernelConsts& kc, cudaStream_t st) {
  const int64_t n = t.n;
  const int nb = nblocks(n, kNT);
  if (prec == kF32)
    GS_CUDA_OK(pdl_launch(k_gather<float>, nb, kNT, 0, st, (const float4*)rec, t.perm.as<int>(), n, kc.kappa, kc.c0[0], kc.c0[1], kc.c0[2], 1, t.srec.as<float4>(), t.squ.as<float4>()));
  else
    GS_CUDA_OK(pdl_launch(k_gather<double>, nb, kNT, 0, st, (const double4*)rec, t.perm.as<int>(), n, kc.kappa, kc.c0[0], kc.c0[1], kc.c0[2], 0, t.srec.as<double4>(), t.squ.as<double4>()));
  GS_CUDA_OK(cudaGetLastError());
  return tree_finalize_fwd(prec, t, kc, st);
}

namespace {
// A single-point leaf's adjoint unit in nadj is the point's own (alpha, beta)
// (k_finalize mode 1): refresh it with the per-point adjoints so that direct
// terms read the new values while the aggregate nodes keep their annotation.
template <typename R>
__global__ void k_leaf_adj(const int4* meta, const int* mp, const V4<R>* sadj, V4<R>* nadj) {
  const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
  if (i >= *mp) return;
  const int4 mi = meta[i];
  if (!((mi.w & 1) && mi.z == mi.y)) return;
  st4(nadj + 2 * i, ld4(sadj + 2 * mi.y));
  st4(nadj + 2 * i + 1, ld4(sadj + 2 * mi.y + 1));
}
}  // namespace

int tree_set_point_adjoints(int prec, DevTree& t, const void* adj, cudaStream_t st) {
  const int64_t n = t.n;
  GS_TRY_INT(t.sadj.ensure(2 * vec_bytes(prec) * n));
  const int nb = nblocks(n, kNT), mb = nblocks(t.cap, kNT);
  const int* mp = t.first.as<int>() + n;
  if (prec == kF32) {
    k_gather_adj<float><<<nb, kNT, 0, st>>>((const float4*)adj, t.perm.as<int>(), n, t.sadj.as<float4>());
    if (t.adj_valid) k_leaf_adj<float><<<mb, kNT, 0, st>>>(t.meta.as<int4>(), mp, t.sadj.as<float4>(), t.nadj.as<float4>());
  } else {
    k_gather_adj<double><<<nb, kNT, 0, st>>>((const double4*)adj, t.perm.as<int>(), n, t.sadj.as<double4>());
    if (t.adj_valid) k_leaf_adj<double><<<mb, kNT, 0, st>>>(t.meta.as<int4>(), mp, t.sadj.as<double4>(), t.nadj.as<double4>());
  }
  GS_CUDA_OK(cudaGetLastError());
  return GS_OK;
}

int tree_accumulate(int prec, DevTree& t, const void* adj, cudaStream_t st) {
  const int64_t n = t.n, cap = t.cap;
  const size_t vb = vec_bytes(prec);
  GS_TRY_INT(t.sadj.ensure(2 * vb * n));
  GS_TRY_INT(t.asum.ensure(sizeof(double4) * cap));
  GS_TRY_INT(t.bsum.ensure(sizeof(double4) * cap));
  GS_TRY_INT(t.nadj.ensure(2 * vb * cap));
  GS_TRY_INT(aggregate(1, prec, t, adj, t.kc, st));
  t.adj_valid = true;
  return GS_OK;
}

namespace {

// single-point leaves' stored fields for a download (k_aggregate leaves them
// out): box = the point, sums = the point, its momentum, alpha and beta
template <typename R>
__global__ void k_fill_leaves(const int4* meta, int64_t m, const V4<R>* squ, const V4<R>* srec,
                              const V4<R>* sadj, V4<R>* lo, V4<R>* hi, double4* psum,
                              double4* msum, double4* asum, double4* bsum) {
  const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
  if (i >= m) return;
  const int4 mi = meta[i];
  if (!((mi.w & 1) && mi.y == mi.z)) return;
  const V4<R> q = ld4(squ + mi.y), p = ld4(srec + 2 * mi.y + 1);
  st4(lo + i, q);
  st4(hi + i, q);
  psum[i] = make_double4(q.x, q.y, q.z, 0);
  msum[i] = make_double4(p.x, p.y, p.z, 0);
  if (asum) {
    const V4<R> al = ld4(sadj + 2 * mi.y), be = ld4(sadj + 2 * mi.y + 1);
    asum[i] = make_double4(al.x, al.y, al.z, 0);
    bsum[i] = make_double4(be.x, be.y, be.z, 0);
  }
}

template <typename R>
__global__ void k_dl_nodes(const int4* meta, const int* parent, int64_t m, const V4<R>* lo,
                           const V4<R>* hi, const double4* psum, const double4* msum,
                           const double4* asum, const double4* bsum, int32_t* level,
                           int32_t* par, int32_t* skip, int32_t* range, double* boxes,
                           double* sums, uint32_t* count) {
  const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
  if (i >= m) return;
  const int4 mi = meta[i];
  if (level) level[i] = mi.w >> 8;
  if (par) par[i] = parent[i];
  if (skip) skip[i] = mi.x;
  if (range) { range[2 * i] = mi.y; range[2 * i + 1] = mi.z; }
  if (count) count[i] = (uint32_t)(mi.z - mi.y + 1);
  if (boxes) {
    const V4<R> l = ld4(lo + i), h = ld4(hi + i);
    boxes[12 * i + 6] = l.x; boxes[12 * i + 7] = l.y; boxes[12 * i + 8] = l.z;
    boxes[12 * i + 9] = h.x; boxes[12 * i + 10] = h.y; boxes[12 * i + 11] = h.z;
  }
  if (sums) {
    const double4 z = make_double4(0, 0, 0, 0);
    const double4 v[4] = {psum[i], msum[i], asum ? asum[i] : z, bsum ? bsum[i] : z};
    for (int k = 0; k < 4; ++k) {
      sums[12 * i + 3 * k] = v[k].x; sums[12 * i + 3 * k + 1] = v[k].y; sums[12 * i + 3 * k + 2] = v[k].z;
    }
  }
}

template <typename T>
int dl(T* host, const DBuf& d, int64_t count, cudaStream_t st) {
  if (host && count > 0)
    GS_CUDA_OK(cudaMemcpyAsync(host, d.ptr, sizeof(T) * count, cudaMemcpyDeviceToHost, st));
  return GS_OK;
}

}  // namespace

int64_t tree_node_count(DevTree& t, cudaStream_t st) {
  if (t.m < 0) {
    int m = 0;
    if (cudaMemcpyAsync(&m, t.first.as<int>() + t.n, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return -1;
    t.m = m;
  }
  return t.m;
}

int tree_download(DevTree& t, cudaStream_t st, int32_t* order, uint64_t* key_hi,
                  uint64_t* key_lo, int32_t* level, int32_t* parent, int32_t* skip,
                  int32_t* range, double* boxes, double* sums, uint32_t* count) {
  const int64_t n = t.n, m = tree_node_count(t, st);
  if (m < 0) return cuda_fail(cudaGetLastError(), "tree_node_count", __FILE__, __LINE__);
  if (m > t.cap) {
    set_error("octree node capacity exceeded (degenerate clustering)");
    return GS_INTERNAL;
  }
  DBuf b_level, b_par, b_skip, b_range, b_boxes, b_sums, b_count;
  if (level) GS_TRY_INT(b_level.ensure(4 * m));
  if (parent) GS_TRY_INT(b_par.ensure(4 * m));
  if (skip) GS_TRY_INT(b_skip.ensure(4 * m));
  if (range) GS_TRY_INT(b_range.ensure(8 * m));
  if (boxes) GS_TRY_INT(b_boxes.ensure(96 * m));
  if (sums) GS_TRY_INT(b_sums.ensure(96 * m));
  if (count) GS_TRY_INT(b_count.ensure(4 * m));
  const int mb = nblocks(m, kNT);
  {  // key_lo (computed lazily by the build: only with equal key_hi neighbours)
    const int nb = nblocks(n, kNT);
    if (t.prec == kF32)
      k_keys_lo_leaf<float><<<nb, kNT, 0, st>>>(t.squ.as<float4>(), t.perm.as<int>(), n, t.root.as<double>(), t.skey_hi.as<uint64_t>(), t.skey_lo.as<uint64_t>(), t.key_lo.as<uint64_t>());
    else
      k_keys_lo_leaf<double><<<nb, kNT, 0, st>>>(t.squ.as<double4>(), t.perm.as<int>(), n, t.root.as<double>(), t.skey_hi.as<uint64_t>(), t.skey_lo.as<uint64_t>(), t.key_lo.as<uint64_t>());
  }
  const double4* as = t.adj_valid ? t.asum.as<double4>() : nullptr;
  const double4* bs = t.adj_valid ? t.bsum.as<double4>() : nullptr;
  if (t.prec == kF32) {
    k_fill_leaves<float><<<mb, kNT, 0, st>>>(t.meta.as<int4>(), m, t.squ.as<float4>(), t.srec.as<float4>(), t.sadj.as<float4>(), t.lo.as<float4>(), t.hi.as<float4>(), t.psum.as<double4>(), t.msum.as<double4>(), (double4*)as, (double4*)bs);
    k_dl_nodes<float><<<mb, kNT, 0, st>>>(t.meta.as<int4>(), t.parent.as<int>(), m, t.lo.as<float4>(), t.hi.as<float4>(), t.psum.as<double4>(), t.msum.as<double4>(), as, bs, b_level.as<int32_t>(), b_par.as<int32_t>(), b_skip.as<int32_t>(), b_range.as<int32_t>(), b_boxes.as<double>(), b_sums.as<double>(), b_count.as<uint32_t>());
  } else {
    k_fill_leaves<double><<<mb, kNT, 0, st>>>(t.meta.as<int4>(), m, t.squ.as<double4>(), t.srec.as<double4>(), t.sadj.as<double4>(), t.lo.as<double4>(), t.hi.as<double4>(), t.psum.as<double4>(), t.msum.as<double4>(), (double4*)as, (double4*)bs);
    k_dl_nodes<double><<<mb, kNT, 0, st>>>(t.meta.as<int4>(), t.parent.as<int>(), m, t.lo.as<double4>(), t.hi.as<double4>(), t.psum.as<double4>(), t.msum.as<double4>(), as, bs, b_level.as<int32_t>(), b_par.as<int32_t>(), b_skip.as<int32_t>(), b_range.as<int32_t>(), b_boxes.as<double>(), b_sums.as<double>(), b_count.as<uint32_t>());
  }
  if (boxes)
    k_cells<<<mb, kNT, 0, st>>>(t.meta.as<int4>(), m, t.skey_hi.as<uint64_t>(), t.skey_lo.as<uint64_t>(), t.root.as<double>(), b_boxes.as<double>());
  GS_CUDA_OK(cudaGetLastError());
  GS_TRY_INT(dl(order, t.perm, n, st));
  GS_TRY_INT(dl(key_hi, t.key_hi, n, st));
  GS_TRY_INT(dl(key_lo, t.key_lo, n, st));
  GS_TRY_INT(dl(level, b_level, m, st));
  GS_TRY_INT(dl(parent, b_par, m, st));
  GS_TRY_INT(dl(skip, b_skip, m, st));
  GS_TRY_INT(dl(range, b_range, 2 * m, st));
  GS_TRY_INT(dl(boxes, b_boxes, 12 * m, st));
  GS_TRY_INT(dl(sums, b_sums, 12 * m, st));
  GS_TRY_INT(dl(count, b_count, m, st));
  GS_CUDA_OK(cudaStreamSynchronize(st));
  return GS_OK;
}

int trace_install_tree(unsigned long long* buf) {
  GS_CUDA_OK(trace_install_here(buf));
  return GS_OK;
}

}  // namespace gsb
