// allpairs.cu -- exact O(N^2) kernel sums on sm_100a (FP32 + FP64).
//
// Replaces kernel_exact.cpp:29-61 (hamiltonian_with_gradients), :70-82
// (exact_velocity) and :84-135 (hessian_products). The reference sweeps the
// upper triangle and scatters every pair to both ends; on the GPU each thread
// OWNS `TPT` targets and gathers over all sources (self included: its terms
// are exactly the reference's explicit diagonal, kernel_exact.cpp:41-44 and
// :94-97), so no atomics and a fixed, launch-independent summation order per
// target -> bitwise-deterministic results (test_shooting.cpp:305-318).
//
// Work decomposition: grid.x = target blocks of NT*TPT targets, grid.y = S
// source chunks; each CTA streams its chunk through shared memory in tiles of
// TILE records (coalesced 16-B loads, broadcast LDS.128 reads) and writes one
// partial per (chunk, target). The stage epilogue (epilogue.cu) folds the S
// partials in fixed order, applies the constants and the integrator update.
// S is picked so that the grid fills an integral number of waves of resident
// CTAs (148 SMs x occupancy).
//
// FP32 inner loop per (target, source) pair, pre-scaled coordinates
// (gs_common.cuh): 3 FADD (d) + FMUL+2 FFMA (-r^2) + MUFU.EX2 (g) + FMUL+2 FFMA
// (p_i.p_j) + FMUL (c) + 3 FFMA (sum g p_j) + 3 FFMA (sum c d) = 16 FP32 + 1 SFU.
// No tensor cores: the contraction dimension is 3.
#include <cstdio>
#include <cstdlib>

#include "engine.h"
#include "gs_exp.cuh"

namespace gsb {

constexpr int kTile = 256;
#ifndef GS_SORTED_UNR
#define GS_SORTED_UNR 8
#endif
#ifndef GS_F64_UNR
#define GS_F64_UNR 4
#endif
#ifndef GS_HESS_MINB
#define GS_HESS_MINB 1
#endif

// ----------------------------------------------------------------------------
// forward RHS partials: A = sum_j g p_j, B = sum_j (p_i.p_j) g d'_ij
// ----------------------------------------------------------------------------
constexpr int kSortedUnr = GS_SORTED_UNR;  // source-loop unroll, k_rhs_f32x2_sorted
constexpr int kF64Unr = GS_F64_UNR;        // source-loop unroll, k_rhs_f64

template <int TPT, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_rhs_f32(const float4* __restrict__ rec, int n,
                                                      int tgt_begin, int n_tgt, int chunk,
                                                      float kap, float kc0x, float kc0y, float kc0z,
                                                      float4* __restrict__ part) {
  __shared__ float4 sq[kTile];
  __shared__ float4 sp[kTile];
  float qx[TPT], qy[TPT], qz[TPT], px[TPT], py[TPT], pz[TPT];
  float ax[TPT], ay[TPT], az[TPT], bx[TPT], by[TPT], bz[TPT];
  const int tb = blockIdx.x * NT * TPT + threadIdx.x;
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int t = tb + k * NT;
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f), p = q;
    if (t < n_tgt) {
      q = rec[2 * (tgt_begin + t)];
      p = rec[2 * (tgt_begin + t) + 1];
    }
    qx[k] = fmaf(kap, q.x, -kc0x); qy[k] = fmaf(kap, q.y, -kc0y); qz[k] = fmaf(kap, q.z, -kc0z);
    px[k] = p.x; py[k] = p.y; pz[k] = p.z;
    ax[k] = ay[k] = az[k] = bx[k] = by[k] = bz[k] = 0.f;
  }
  const int j0 = blockIdx.y * chunk;
  const int j1 = min(n, j0 + chunk);
  for (int jt = j0; jt < j1; jt += kTile) {
    __syncthreads();
    for (int u = threadIdx.x; u < kTile; u += NT) {
      const int j = jt + u;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f), p = q;
      if (j < j1) {
        q = rec[2 * j];
        p = rec[2 * j + 1];
        q = make_float4(fmaf(kap, q.x, -kc0x), fmaf(kap, q.y, -kc0y), fmaf(kap, q.z, -kc0z), 0.f);
      }
      sq[u] = q;  // zero records contribute exactly 0 (p = 0)
      sp[u] = p;
    }
    __syncthreads();
    // all TPT exponentials are issued before the first one is consumed, so
    // the MUFU latency hides behind independent work of the same warp
#pragma unroll 2
    for (int u = 0; u < kTile; ++u) {
      const float4 a = sq[u];
      const float4 b = sp[u];
      float dx[TPT], dy[TPT], dz[TPT], g[TPT];
#pragma unroll
      for (int k = 0; k < TPT; ++k) {
        dx[k] = qx[k] - a.x; dy[k] = qy[k] - a.y; dz[k] = qz[k] - a.z;
        float nr2 = -dx[k] * dx[k];
        nr2 = fmaf(-dy[k], dy[k], nr2);
        nr2 = fmaf(-dz[k], dz[k], nr2);
        g[k] = ex2(nr2);
      }
#pragma unroll
      for (int k = 0; k < TPT; ++k) {
        float pp = px[k] * b.x;
        pp = fmaf(py[k], b.y, pp);
        pp = fmaf(pz[k], b.z, pp);
        const float c = pp * g[k];
        ax[k] = fmaf(g[k], b.x, ax[k]);
        ay[k] = fmaf(g[k], b.y, ay[k]);
        az[k] = fmaf(g[k], b.z, az[k]);
        bx[k] = fmaf(c, dx[k], bx[k]);
        by[k] = fmaf(c, dy[k], by[k]);
        bz[k] = fmaf(c, dz[k], bz[k]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int t = tb + k * NT;
    if (t < n_tgt) {
      float4* o = part + 2 * ((size_t)blockIdx.y * n_tgt + t);
      o[0] = make_float4(ax[k], ay[k], az[k], 0.f);
      o[1] = make_float4(bx[k], by[k], bz[k], 0.f);
    }
  }
}

// packed FP32x2 arithmetic (f2, sub2, mul2, fma2, ...): gs_common.cuh

// Packed variant of k_rhs_f32: TPT targets per thread as TPT/2 register
// pairs. Per two (target, source) pairs: 3 FADD2 + FMUL2 + 2 FFMA2 (r^2) +
// 2 MUFU + FMUL2 + 2 FFMA2 (p_i.p_j) + FMUL2 (c) + 3 FFMA2 (sum g p_j) +
// 3 FFMA2 (sum c d') = 16 packed FP32 + 2 SFU issue slots (9 per pair instead
// of 17); identical arithmetic per target to the scalar kernel.
template <int TPT, int NT, int MINB, int UNR = 2>
__global__ void __launch_bounds__(NT, MINB) k_rhs_f32x2(const float4* __restrict__ rec, int n,
                                                        int tgt_begin, int n_tgt, int chunk,
                                                        float kap, float kc0x, float kc0y,
                                                        float kc0z, float4* __restrict__ part) {
  constexpr int TP = TPT / 2;
  __shared__ float4 sq[kTile];
  __shared__ float4 sp[kTile];
  f2 qx[TP], qy[TP], qz[TP], px[TP], py[TP], pz[TP];
  f2 ax[TP], ay[TP], az[TP], bx[TP], by[TP], bz[TP];
  const int tb = blockIdx.x * NT * TPT + threadIdx.x;
#pragma unroll
  for (int k = 0; k < TP; ++k) {
    float4 q[2], p[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = tb + (2 * k + h) * NT;
      q[h] = make_float4(0.f, 0.f, 0.f, 0.f);
      p[h] = q[h];
      if (t < n_tgt) {
        q[h] = rec[2 * (tgt_begin + t)];
        p[h] = rec[2 * (tgt_begin + t) + 1];
      }
      q[h] = make_float4(fmaf(kap, q[h].x, -kc0x), fmaf(kap, q[h].y, -kc0y), fmaf(kap, q[h].z, -kc0z), 0.f);
    }
    qx[k] = pk2(q[0].x, q[1].x); qy[k] = pk2(q[0].y, q[1].y); qz[k] = pk2(q[0].z, q[1].z);
    px[k] = pk2(p[0].x, p[1].x); py[k] = pk2(p[0].y, p[1].y); pz[k] = pk2(p[0].z, p[1].z);
    ax[k] = ay[k] = az[k] = bx[k] = by[k] = bz[k] = pk2(0.f, 0.f);
  }
  const int j0 = blockIdx.y * chunk;
  const int j1 = min(n, j0 + chunk);
  for (int jt = j0; jt < j1; jt += kTile) {
    __syncthreads();
    for (int u = threadIdx.x; u < kTile; u += NT) {
      const int j = jt + u;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f), p = q;
      if (j < j1) {
        q = rec[2 * j];
        p = rec[2 * j + 1];
        q = make_float4(fmaf(kap, q.x, -kc0x), fmaf(kap, q.y, -kc0y), fmaf(kap, q.z, -kc0z), 0.f);
      }
      sq[u] = q;  // zero records contribute exactly 0 (p = 0)
      sp[u] = p;
    }
    __syncthreads();
#pragma unroll UNR
    for (int u = 0; u < kTile; ++u) {
      const float4 a = sq[u];
      const float4 b = sp[u];
      const f2 axx = bc2(a.x), ayy = bc2(a.y), azz = bc2(a.z);
      const f2 bxx = bc2(b.x), byy = bc2(b.y), bzz = bc2(b.z);
      f2 dx[TP], dy[TP], dz[TP], g[TP];
#pragma unroll
      for (int k = 0; k < TP; ++k) {
        dx[k] = sub2(qx[k], axx);
        dy[k] = sub2(qy[k], ayy);
        dz[k] = sub2(qz[k], azz);
        f2 r2 = mul2(dx[k], dx[k]);
        r2 = fma2(dy[k], dy[k], r2);
        r2 = fma2(dz[k], dz[k], r2);
        g[k] = nex2x2(r2);
      }
#pragma unroll
      for (int k = 0; k < TP; ++k) {
        f2 pp = mul2(px[k], bxx);
        pp = fma2(py[k], byy, pp);
        pp = fma2(pz[k], bzz, pp);
        const f2 c = mul2(pp, g[k]);
        ax[k] = fma2(g[k], bxx, ax[k]);
        ay[k] = fma2(g[k], byy, ay[k]);
        az[k] = fma2(g[k], bzz, az[k]);
        bx[k] = fma2(c, dx[k], bx[k]);
        by[k] = fma2(c, dy[k], by[k]);
        bz[k] = fma2(c, dz[k], bz[k]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < TP; ++k) {
    float a0[2][3], b0[2][3];
    up2(ax[k], a0[0][0], a0[1][0]); up2(ay[k], a0[0][1], a0[1][1]); up2(az[k], a0[0][2], a0[1][2]);
    up2(bx[k], b0[0][0], b0[1][0]); up2(by[k], b0[0][1], b0[1][1]); up2(bz[k], b0[0][2], b0[1][2]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = tb + (2 * k + h) * NT;
      if (t < n_tgt) {
        float4* o = part + 2 * ((size_t)blockIdx.y * n_tgt + t);
        o[0] = make_float4(a0[h][0], a0[h][1], a0[h][2], 0.f);
        o[1] = make_float4(b0[h][0], b0[h][1], b0[h][2], 0.f);
      }
    }
  }
}

// ---- symmetric exact FP32 RHS: every unordered pair evaluated once ----------
// The reference sweeps i < j and scatters each pair to both ends
// (kernel_exact.cpp:29-61); this kernel does the same at tile granularity.
// The n points form T tiles of NT*TPT; CTA (I, k) evaluates the unordered
// tile pair {I, J = (I + k) mod T}, k = 0 .. floor(T/2) (for even T the
// k = T/2 pairs belong to I < T/2 only), so every unordered tile pair is
// taken exactly once. Threads own TPT targets of tile I in registers (packed
// pairs, as k_rhs_f32x2) and stream the sources of tile J through shared
// memory; g, c = g p_i.p_j and d_ij of a pair are computed once and feed
// BOTH ends:
//   i side (registers):  A_i += g p_j,  B_i += c d_ij
//   j side (shared):     A_j += g p_i,  B_j -= c d_ij
// Per two unordered pairs (a packed target pair x one source): 22 packed FP32
// + 2 MUFU issue slots = 6 per ordered pair (k_rhs_f32x2: 9).
// The j side needs no atomics: at step s of a 32-source batch lane l takes
// source (l + s) mod 32, so the 32 lanes of a warp always hold 32 distinct
// sources, and the source's packed j accumulators travel with it from lane to
// lane (lane l takes them over from lane l + 1 by one shuffle per accumulator
// and step; round 2 first used a fold + shared read-modify-write per step:
// 4 % slower at 1M, 8 % at 100k). After 32 steps every lane holds one source's
// sums over the warp's 32 x TPT targets, folded over the packed halves into
// the warp's copy of the j accumulators, summed in warp order after the
// sub-tile.
// Partials: target t of tile X receives exactly T partials, one per tile Y
// (slot Y): the i side of the pair (X, Y), the j side of the pair (Y, X), or,
// for Y = X, the diagonal pair evaluated gather-style (ordered pairs, self
// included: the reference's explicit diagonal term). The epilogue folds the
// T slots in fixed order, so results are deterministic (bitwise repeatable).
#ifndef GS_SYM_UNR
#define GS_SYM_UNR 4
#endif
template <int TPT, int NT, int MINB, int SB, int SYM_UNR = GS_SYM_UNR>
__global__ void __launch_bounds__(NT, MINB)
    k_rhs_sym_f32x2(const float4* __restrict__ rec, int n, int T, float kap, float kc0x,
                    float kc0y, float kc0z, float4* __restrict__ part, int row0 = 0,
                    int k0 = -1) {
  constexpr int TP = TPT / 2, TILE = NT * TPT, NW = NT / 32;
  static_assert(TILE % SB == 0 && SB % 32 == 0 && TPT % 2 == 0, "tile shape");
  __shared__ float4 sq[SB];
  __shared__ float4 sp[SB];
  __shared__ float2 sj[NW][3][SB];
  // row0: multi-GPU rows (rhs_sym_rows). k0 >= 0: diagonal group [k0, k0 +
  // gridDim.y) of a problem whose T tile slots would not fit (rhs_sym_partials):
  // the i side goes to slot 2(k - k0), the j side to 2(k - k0) + 1 (the
  // layout of k_rhs_sym_f64), folded into a running sum by k_fold_group_f32
  const int I = row0 + blockIdx.x, k = (k0 < 0 ? 0 : k0) + blockIdx.y;
  const int J = I + k < T ? I + k : I + k - T;
  const size_t slot_i = k0 < 0 ? (size_t)J : (size_t)(2 * (k - k0));
  const size_t slot_j = k0 < 0 ? (size_t)I : (size_t)(2 * (k - k0) + 1);
  if (2 * k == T && I >= k) {  // even T: the pair {I, I + T/2} once
    if (k0 >= 0) {  // grouped: zeros in the two slots this CTA leaves empty
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int u = threadIdx.x; u < TILE; u += NT) {
        const int t = I * TILE + u, j = J * TILE + u;
        if (t < n) part[2 * (slot_i * n + t)] = part[2 * (slot_i * n + t) + 1] = z;
        if (j < n) part[2 * (slot_j * n + j)] = part[2 * (slot_j * n + j) + 1] = z;
      }
    }
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  f2 qx[TP], qy[TP], qz[TP], px[TP], py[TP], pz[TP];
  f2 ax[TP], ay[TP], az[TP], bx[TP], by[TP], bz[TP];
  const int tb = I * TILE + threadIdx.x;
#pragma unroll
  for (int kk = 0; kk < TP; ++kk) {
    float4 q[2], p[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = tb + (2 * kk + h) * NT;
      q[h] = make_float4(0.f, 0.f, 0.f, 0.f);
      p[h] = q[h];
      if (t < n) {
        q[h] = rec[2 * t];
        p[h] = rec[2 * t + 1];
      }
      q[h] = make_float4(fmaf(kap, q[h].x, -kc0x), fmaf(kap, q[h].y, -kc0y), fmaf(kap, q[h].z, -kc0z), 0.f);
    }
    qx[kk] = pk2(q[0].x, q[1].x); qy[kk] = pk2(q[0].y, q[1].y); qz[kk] = pk2(q[0].z, q[1].z);
    px[kk] = pk2(p[0].x, p[1].x); py[kk] = pk2(p[0].y, p[1].y); pz[kk] = pk2(p[0].z, p[1].z);
    ax[kk] = ay[kk] = az[kk] = bx[kk] = by[kk] = bz[kk] = pk2(0.f, 0.f);
  }
  const int jbase = J * TILE;
  for (int st = 0; st < TILE; st += SB) {
    __syncthreads();
    for (int u = threadIdx.x; u < SB; u += NT) {
      const int j = jbase + st + u;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f), p = q;
      if (j < n) {
        q = rec[2 * j];
        p = rec[2 * j + 1];
        q = make_float4(fmaf(kap, q.x, -kc0x), fmaf(kap, q.y, -kc0y), fmaf(kap, q.z, -kc0z), 0.f);
      }
      sq[u] = q;  // zero records contribute exactly 0 (p = 0)
      sp[u] = p;
    }
    __syncthreads();
    if (k == 0) {
      // diagonal tile pair: gather over the tile's own points (ordered pairs)
#pragma unroll 4
      for (int u = 0; u < SB; ++u) {
        const float4 a = sq[u];
        const float4 b = sp[u];
        const f2 axx = bc2(a.x), ayy = bc2(a.y), azz = bc2(a.z);
        const f2 bxx = bc2(b.x), byy = bc2(b.y), bzz = bc2(b.z);
        f2 dx[TP], dy[TP], dz[TP], g[TP];
#pragma unroll
        for (int kk = 0; kk < TP; ++kk) {
          dx[kk] = sub2(qx[kk], axx);
          dy[kk] = sub2(qy[kk], ayy);
          dz[kk] = sub2(qz[kk], azz);
          f2 r2 = mul2(dx[kk], dx[kk]);
          r2 = fma2(dy[kk], dy[kk], r2);
          r2 = fma2(dz[kk], dz[kk], r2);
          g[kk] = nex2x2(r2);
        }
#pragma unroll
        for (int kk = 0; kk < TP; ++kk) {
          f2 pp = mul2(px[kk], bxx);
          pp = fma2(py[kk], byy, pp);
          pp = fma2(pz[kk], bzz, pp);
          const f2 c = mul2(pp, g[kk]);
          ax[kk] = fma2(g[kk], bxx, ax[kk]);
          ay[kk] = fma2(g[kk], byy, ay[kk]);
          az[kk] = fma2(g[kk], bzz, az[kk]);
          bx[kk] = fma2(c, dx[kk], bx[kk]);
          by[kk] = fma2(c, dy[kk], by[kk]);
          bz[kk] = fma2(c, dz[kk], bz[kk]);
        }
      }
      continue;
    }
    float2* sj0 = sj[warp][0];
    float2* sj1 = sj[warp][1];
    float2* sj2 = sj[warp][2];
    for (int b0 = 0; b0 < SB; b0 += 32) {
      // the packed j accumulators of source (lane + s) mod 32 travel with it
      // from lane to lane: one 64-bit shuffle per accumulator and step, no
      // fold and no shared read-modify-write inside the loop
      f2 tax = pk2(0.f, 0.f), tay = tax, taz = tax, tbx = tax, tby = tax, tbz = tax;
#pragma unroll SYM_UNR
      for (int s = 0; s < 32; ++s) {
        const int u = b0 + ((lane + s) & 31);
        const float4 a = sq[u];
        const float4 b = sp[u];
        const f2 axx = bc2(a.x), ayy = bc2(a.y), azz = bc2(a.z);
        const f2 bxx = bc2(b.x), byy = bc2(b.y), bzz = bc2(b.z);
        f2 dx[TP], dy[TP], dz[TP], g[TP];
#pragma unroll
        for (int kk = 0; kk < TP; ++kk) {
          dx[kk] = sub2(qx[kk], axx);
          dy[kk] = sub2(qy[kk], ayy);
          dz[kk] = sub2(qz[kk], azz);
          f2 r2 = mul2(dx[kk], dx[kk]);
          r2 = fma2(dy[kk], dy[kk], r2);
          r2 = fma2(dz[kk], dz[kk], r2);
          g[kk] = nex2x2(r2);
        }
#pragma unroll
        for (int kk = 0; kk < TP; ++kk) {
          f2 pp = mul2(px[kk], bxx);
          pp = fma2(py[kk], byy, pp);
          pp = fma2(pz[kk], bzz, pp);
          const f2 c = mul2(pp, g[kk]);
          ax[kk] = fma2(g[kk], bxx, ax[kk]);
          ay[kk] = fma2(g[kk], byy, ay[kk]);
          az[kk] = fma2(g[kk], bzz, az[kk]);
          bx[kk] = fma2(c, dx[kk], bx[kk]);
          by[kk] = fma2(c, dy[kk], by[kk]);
          bz[kk] = fma2(c, dz[kk], bz[kk]);
          tax = fma2(g[kk], px[kk], tax); tay = fma2(g[kk], py[kk], tay);
          taz = fma2(g[kk], pz[kk], taz);
          tbx = fma2(c, dx[kk], tbx); tby = fma2(c, dy[kk], tby); tbz = fma2(c, dz[kk], tbz);
        }
        // lane l takes over the sums of source (l + 1 + s) mod 32 from lane l + 1
        const int from = (lane + 1) & 31;
        tax.v = __shfl_sync(0xffffffffu, tax.v, from); tay.v = __shfl_sync(0xffffffffu, tay.v, from);
        taz.v = __shfl_sync(0xffffffffu, taz.v, from); tbx.v = __shfl_sync(0xffffffffu, tbx.v, from);
        tby.v = __shfl_sync(0xffffffffu, tby.v, from); tbz.v = __shfl_sync(0xffffffffu, tbz.v, from);
      }
      {  // after 32 steps lane l holds source l's sums over all 32 lanes
        float l0, h0, l1, h1;
        const int u = b0 + lane;
        up2(tax, l0, h0); up2(tay, l1, h1); sj0[u] = make_float2(l0 + h0, l1 + h1);
        up2(taz, l0, h0); up2(tbx, l1, h1); sj1[u] = make_float2(l0 + h0, l1 + h1);
        up2(tby, l0, h0); up2(tbz, l1, h1); sj2[u] = make_float2(l0 + h0, l1 + h1);
      }
    }
    __syncthreads();
    // j side of this sub-tile's sources: the warp copies in warp order, slot I
    for (int u = threadIdx.x; u < SB; u += NT) {
      const int j = jbase + st + u;
      if (j < n) {
        float2 s0 = sj[0][0][u], s1 = sj[0][1][u], s2 = sj[0][2][u];
#pragma unroll
        for (int w = 1; w < NW; ++w) {
          const float2 t0 = sj[w][0][u], t1 = sj[w][1][u], t2 = sj[w][2][u];
          s0.x += t0.x; s0.y += t0.y; s1.x += t1.x; s1.y += t1.y; s2.x += t2.x; s2.y += t2.y;
        }
        float4* o = part + 2 * (slot_j * n + j);
        o[0] = make_float4(s0.x, s0.y, s1.x, 0.f);
        o[1] = make_float4(-s1.y, -s2.x, -s2.y, 0.f);
      }
    }
  }
  // i side: slot J (the diagonal pair: J = I)
#pragma unroll
  for (int kk = 0; kk < TP; ++kk) {
    float a0[2][3], b0[2][3];
    up2(ax[kk], a0[0][0], a0[1][0]); up2(ay[kk], a0[0][1], a0[1][1]); up2(az[kk], a0[0][2], a0[1][2]);
    up2(bx[kk], b0[0][0], b0[1][0]); up2(by[kk], b0[0][1], b0[1][1]); up2(bz[kk], b0[0][2], b0[1][2]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = tb + (2 * kk + h) * NT;
      if (t < n) {
        float4* o = part + 2 * (slot_i * n + t);
        o[0] = make_float4(a0[h][0], a0[h][1], a0[h][2], 0.f);
        o[1] = make_float4(b0[h][0], b0[h][1], b0[h][2], 0.f);
        if (k0 >= 0 && k == 0) {  // grouped diagonal: its j slot is zero
          float4* z = part + 2 * (slot_j * n + t);
          z[0] = z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
  }
}

// acc[t] (+)= sum over a diagonal group's S slots of part[s][t] (4 float4 per
// target: the Hessian products), in slot order
__global__ void k_fold_group4_f32(const float4* __restrict__ part, int S, int n, int first,
                                  float4* __restrict__ acc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  for (int c = 0; c < 4; ++c) {
    float4 a = first ? make_float4(0.f, 0.f, 0.f, 0.f) : acc[4 * t + c];
    for (int s = 0; s < S; ++s) {
      const float4 x = part[4 * ((size_t)s * n + t) + c];
      a.x += x.x; a.y += x.y; a.z += x.z;
    }
    acc[4 * t + c] = a;
  }
}

// acc[t] (+)= sum over a diagonal group's S slots of part[s][t], in slot order
__global__ void k_fold_group_f32(const float4* __restrict__ part, int S, int n, int first,
                                 float4* __restrict__ acc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  float4 a = first ? make_float4(0.f, 0.f, 0.f, 0.f) : acc[2 * t];
  float4 b = first ? make_float4(0.f, 0.f, 0.f, 0.f) : acc[2 * t + 1];
  for (int s = 0; s < S; ++s) {
    const float4 x = part[2 * ((size_t)s * n + t)], y = part[2 * ((size_t)s * n + t) + 1];
    a.x += x.x; a.y += x.y; a.z += x.z;
    b.x += y.x; b.y += y.y; b.z += y.z;
  }
  acc[2 * t] = a;
  acc[2 * t + 1] = b;
}

// ---- exact RHS in Morton order with the FP32 underflow cutoff -----------------
// Same packed arithmetic as k_rhs_f32x2, but targets and sources are the
// points in Morton (leaf) order (t.srec: interaction coordinates already
// scaled, p), so a CTA's 1024 targets and a 256-source tile each occupy a small
// box. If the two boxes are farther apart than cut2 (scaled units: every pair
// has -r'^2 <= -cut2 < -150), every weight 2^(-r'^2) of the tile is exactly
// 0 in FP32 (ex2.approx.ftz flushes below 2^-126; 2^-150 rounds to 0), so
// every term the tile would add is +-0 and the accumulators (never -0) are
// unchanged bit for bit: the tile is skipped. With cut2 = +inf nothing is
// skipped; the two runs are bitwise identical (tests/test_gpu_exact.py).
// Partials are written by point index (perm) for the usual epilogue.
template <int TPT, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB)
    k_rhs_f32x2_sorted(const float4* __restrict__ srec, const int* __restrict__ perm, int n,
                       int chunk, const float4* __restrict__ tbox, const float4* __restrict__ sbox,
                       float cut2, float4* __restrict__ part, unsigned long long* cnt) {
  constexpr int TP = TPT / 2;
  __shared__ float4 sq[kTile];
  __shared__ float4 sp[kTile];
  f2 qx[TP], qy[TP], qz[TP], px[TP], py[TP], pz[TP];
  f2 ax[TP], ay[TP], az[TP], bx[TP], by[TP], bz[TP];
  // each warp owns 32 * TPT consecutive (Morton-adjacent) targets, so its box
  // is the 256-point group box sbox[blockIdx.x * NT / 32 + warp] (32 * TPT = kTile)
  static_assert(32 * TPT == kTile, "warp target group = source tile size");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tb = blockIdx.x * NT * TPT + warp * 32 * TPT + lane;
#pragma unroll
  for (int k = 0; k < TP; ++k) {
    float4 q[2], p[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = tb + (2 * k + h) * 32;
      q[h] = make_float4(0.f, 0.f, 0.f, 0.f);
      p[h] = q[h];
      if (t < n) {
        q[h] = srec[2 * t];
        p[h] = srec[2 * t + 1];
      }
    }
    qx[k] = pk2(q[0].x, q[1].x); qy[k] = pk2(q[0].y, q[1].y); qz[k] = pk2(q[0].z, q[1].z);
    px[k] = pk2(p[0].x, p[1].x); py[k] = pk2(p[0].y, p[1].y); pz[k] = pk2(p[0].z, p[1].z);
    ax[k] = ay[k] = az[k] = bx[k] = by[k] = bz[k] = pk2(0.f, 0.f);
  }
  const float4 tl = tbox[2 * blockIdx.x], th = tbox[2 * blockIdx.x + 1];
  const int wg = blockIdx.x * (NT / 32) + warp;
  const bool wvalid = wg * kTile < n;
  const float4 wl = wvalid ? sbox[2 * wg] : tl, wh = wvalid ? sbox[2 * wg + 1] : th;
  const int j0 = blockIdx.y * chunk;
  const int j1 = min(n, j0 + chunk);
  for (int jt = j0; jt < j1; jt += kTile) {
    const float4 sl = sbox[2 * (jt / kTile)], sh = sbox[2 * (jt / kTile) + 1];
    const float gx = fmaxf(0.f, fmaxf(sl.x - th.x, tl.x - sh.x));
    const float gy = fmaxf(0.f, fmaxf(sl.y - th.y, tl.y - sh.y));
    const float gz = fmaxf(0.f, fmaxf(sl.z - th.z, tl.z - sh.z));
    if (gx * gx + gy * gy + gz * gz > cut2) continue;  // CTA-uniform: every weight is 0
    __syncthreads();
    for (int u = threadIdx.x; u < kTile; u += NT) {
      const int j = jt + u;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f), p = q;
      if (j < j1) {
        q = srec[2 * j];
        p = srec[2 * j + 1];
      }
      sq[u] = q;  // zero records contribute exactly 0 (p = 0)
      sp[u] = p;
    }
    __syncthreads();
    {  // the same test on this warp's own box: warp-uniform skip of the compute
      const float hx = fmaxf(0.f, fmaxf(sl.x - wh.x, wl.x - sh.x));
      const float hy = fmaxf(0.f, fmaxf(sl.y - wh.y, wl.y - sh.y));
      const float hz = fmaxf(0.f, fmaxf(sl.z - wh.z, wl.z - sh.z));
      if (!wvalid || hx * hx + hy * hy + hz * hz > cut2) continue;
    }
    if (cnt && lane == 0) atomicAdd(cnt, 1ull);  // GS_EXACT_CUT_DEBUG: computed (warp, tile) pairs
#pragma unroll kSortedUnr
    for (int u = 0; u < kTile; ++u) {
      const float4 a = sq[u];
      const float4 b = sp[u];
      const f2 axx = bc2(a.x), ayy = bc2(a.y), azz = bc2(a.z);
      const f2 bxx = bc2(b.x), byy = bc2(b.y), bzz = bc2(b.z);
      f2 dx[TP], dy[TP], dz[TP], g[TP];
#pragma unroll
      for (int k = 0; k < TP; ++k) {
        dx[k] = sub2(qx[k], axx);
        dy[k] = sub2(qy[k], ayy);
        dz[k] = sub2(qz[k], azz);
        f2 r2 = mul2(dx[k], dx[k]);
        r2 = fma2(dy[k], dy[k], r2);
        r2 = fma2(dz[k], dz[k], r2);
        g[k] = nex2x2(r2);
      }
#pragma unroll
      for (int k = 0; k < TP; ++k) {
        f2 pp = mul2(px[k], bxx);
        pp = fma2(py[k], byy, pp);
        pp = fma2(pz[k], bzz, pp);
        const f2 c = mul2(pp, g[k]);
        ax[k] = fma2(g[k], bxx, ax[k]);
        ay[k] = fma2(g[k], byy, ay[k]);
        az[k] = fma2(g[k], bzz, az[k]);
        bx[k] = fma2(c, dx[k], bx[k]);
        by[k] = fma2(c, dy[k], by[k]);
        bz[k] = fma2(c, dz[k], bz[k]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < TP; ++k) {
    float a0[2][3], b0[2][3];
    up2(ax[k], a0[0][0], a0[1][0]); up2(ay[k], a0[0][1], a0[1][1]); up2(az[k], a0[0][2], a0[1][2]);
    up2(bx[k], b0[0][0], b0[1][0]); up2(by[k], b0[0][1], b0[1][1]); up2(bz[k], b0[0][2], b0[1][2]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = tb + (2 * k + h) * 32;
      if (t < n) {
        float4* o = part + 2 * ((size_t)blockIdx.y * n + perm[t]);
        o[0] = make_float4(a0[h][0], a0[h][1], a0[h][2], 0.f);
        o[1] = make_float4(b0[h][0], b0[h][1], b0[h][2], 0.f);
      }
    }
  }
}

// Tight boxes of consecutive groups of `group` points of srec (lo, hi per group).
__global__ void __launch_bounds__(256) k_group_boxes(const float4* __restrict__ srec, int n,
                                                     int group, float4* __restrict__ box) {
  __shared__ float red[6][8];
  const int g0 = blockIdx.x * group, g1 = min(n, g0 + group);
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int j = g0 + threadIdx.x; j < g1; j += 256) {
    const float4 q = srec[2 * j];
    lo[0] = fminf(lo[0], q.x); lo[1] = fminf(lo[1], q.y); lo[2] = fminf(lo[2], q.z);
    hi[0] = fmaxf(hi[0], q.x); hi[1] = fmaxf(hi[1], q.y); hi[2] = fmaxf(hi[2], q.z);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
    for (int a = 0; a < 3; ++a) { red[a][w] = lo[a]; red[3 + a][w] = hi[a]; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int v = 1; v < 8; ++v)
      for (int a = 0; a < 3; ++a) {
        red[a][0] = fminf(red[a][0], red[a][v]);
        red[3 + a][0] = fmaxf(red[3 + a][0], red[3 + a][v]);
      }
    box[2 * blockIdx.x] = make_float4(red[0][0], red[1][0], red[2][0], 0.f);
    box[2 * blockIdx.x + 1] = make_float4(red[3][0], red[4][0], red[5][0], 0.f);
  }
}

// Packed (FFMA2) Hessian-product kernel: TPT targets as TPT/2 pairs; 40
// packed FP32 + 2 MUFU issue slots per two (target, source) pairs.
template <int TPT, int NT>
__global__ void __launch_bounds__(NT, GS_HESS_MINB) k_hess_f32x2(const float4* __restrict__ rec,
                                                   const float4* __restrict__ adj, int n,
                                                   int tgt_begin, int n_tgt, int chunk, float kap,
                                                   float kc0x, float kc0y, float kc0z, float c1,
                                                   float4* __restrict__ part) {
  constexpr int TP = TPT / 2;
  constexpr int tile = kTile / 2;
  __shared__ float4 sq[tile], sp[tile], sa[tile], sb[tile];
  f2 qx[TP], qy[TP], qz[TP], px[TP], py[TP], pz[TP];
  f2 ix[TP], iy[TP], iz[TP], jx[TP], jy[TP], jz[TP];  // alpha_i, beta_i
  f2 A[TP][12];
  const int tb = blockIdx.x * NT * TPT + threadIdx.x;
#pragma unroll
  for (int k = 0; k < TP; ++k) {
    float4 q[2], p[2], al[2], be[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = tb + (2 * k + h) * NT;
      q[h] = p[h] = al[h] = be[h] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < n_tgt) {
        const int i = tgt_begin + t;
        q[h] = rec[2 * i]; p[h] = rec[2 * i + 1]; al[h] = adj[2 * i]; be[h] = adj[2 * i + 1];
      }
      q[h] = make_float4(fmaf(kap, q[h].x, -kc0x), fmaf(kap, q[h].y, -kc0y), fmaf(kap, q[h].z, -kc0z), 0.f);
    }
    qx[k] = pk2(q[0].x, q[1].x); qy[k] = pk2(q[0].y, q[1].y); qz[k] = pk2(q[0].z, q[1].z);
    px[k] = pk2(p[0].x, p[1].x); py[k] = pk2(p[0].y, p[1].y); pz[k] = pk2(p[0].z, p[1].z);
    ix[k] = pk2(al[0].x, al[1].x); iy[k] = pk2(al[0].y, al[1].y); iz[k] = pk2(al[0].z, al[1].z);
    jx[k] = pk2(be[0].x, be[1].x); jy[k] = pk2(be[0].y, be[1].y); jz[k] = pk2(be[0].z, be[1].z);
#pragma unroll
    for (int c = 0; c < 12; ++c) A[k][c] = pk2(0.f, 0.f);
  }
  const f2 cc1 = bc2(-c1);
  const int j0 = blockIdx.y * chunk;
  const int j1 = min(n, j0 + chunk);
  for (int jt = j0; jt < j1; jt += tile) {
    __syncthreads();
    for (int u = threadIdx.x; u < tile; u += NT) {
      const int j = jt + u;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f), p = q, a = q, b = q;
      if (j < j1) {
        q = rec[2 * j]; p = rec[2 * j + 1]; a = adj[2 * j]; b = adj[2 * j + 1];
        q = make_float4(fmaf(kap, q.x, -kc0x), fmaf(kap, q.y, -kc0y), fmaf(kap, q.z, -kc0z), 0.f);
      }
      sq[u] = q; sp[u] = p; sa[u] = a; sb[u] = b;  // zero records contribute exactly 0
    }
    __syncthreads();
#pragma unroll 1
    for (int u = 0; u < tile; ++u) {
      const float4 Q = sq[u], P = sp[u], Al = sa[u], Be = sb[u];
      const f2 Qx = bc2(Q.x), Qy = bc2(Q.y), Qz = bc2(Q.z);
      const f2 Px = bc2(P.x), Py = bc2(P.y), Pz = bc2(P.z);
      const f2 Ax = bc2(Al.x), Ay = bc2(Al.y), Az = bc2(Al.z);
      const f2 Bx = bc2(Be.x), By = bc2(Be.y), Bz = bc2(Be.z);
#pragma unroll
      for (int k = 0; k < TP; ++k) {
        const f2 dx = sub2(qx[k], Qx), dy = sub2(qy[k], Qy), dz = sub2(qz[k], Qz);
        f2 r2 = mul2(dx, dx);
        r2 = fma2(dy, dy, r2);
        r2 = fma2(dz, dz, r2);
        const f2 g = nex2x2(r2);
        // negated db = beta_j - beta_i, so z = uu d - db is one FFMA2 per axis;
        // the sign comes back through -c1 and the final negation of A[9..11]
        const f2 dbx = sub2(Bx, jx[k]), dby = sub2(By, jy[k]), dbz = sub2(Bz, jz[k]);
        f2 ddb = mul2(dx, dbx);
        ddb = fma2(dy, dby, ddb);
        ddb = fma2(dz, dbz, ddb);
        f2 s1 = mul2(ix[k], Px);
        s1 = fma2(iy[k], Py, s1);
        s1 = fma2(iz[k], Pz, s1);
        s1 = fma2(px[k], Ax, s1);
        s1 = fma2(py[k], Ay, s1);
        s1 = fma2(pz[k], Az, s1);
        f2 pp = mul2(px[k], Px);
        pp = fma2(py[k], Py, pp);
        pp = fma2(pz[k], Pz, pp);
        const f2 t1 = mul2(g, s1);
        A[k][0] = fma2(t1, dx, A[k][0]); A[k][1] = fma2(t1, dy, A[k][1]); A[k][2] = fma2(t1, dz, A[k][2]);
        A[k][3] = fma2(g, Ax, A[k][3]); A[k][4] = fma2(g, Ay, A[k][4]); A[k][5] = fma2(g, Az, A[k][5]);
        const f2 w = mul2(g, pp);
        const f2 uu = mul2(ddb, cc1);  // cc1 = -c1
        const f2 zx = fma2(uu, dx, dbx), zy = fma2(uu, dy, dby), zz = fma2(uu, dz, dbz);
        A[k][6] = fma2(w, zx, A[k][6]); A[k][7] = fma2(w, zy, A[k][7]); A[k][8] = fma2(w, zz, A[k][8]);
        const f2 m = mul2(g, ddb);
        A[k][9] = fma2(m, Px, A[k][9]); A[k][10] = fma2(m, Py, A[k][10]); A[k][11] = fma2(m, Pz, A[k][11]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < TP; ++k) {
    float v[2][12];
#pragma unroll
    for (int c = 0; c < 12; ++c) up2(A[k][c], v[0][c], v[1][c]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = tb + (2 * k + h) * NT;
      if (t < n_tgt) {
        float4* o = part + 4 * ((size_t)blockIdx.y * n_tgt + t);
        o[0] = make_float4(v[h][0], v[h][1], v[h][2], 0.f);
        o[1] = make_float4(v[h][3], v[h][4], v[h][5], 0.f);
        o[2] = make_float4(v[h][6], v[h][7], v[h][8], 0.f);
        o[3] = make_float4(-v[h][9], -v[h][10], -v[h][11], 0.f);
      }
    }
  }
}

// Symmetric Hessian-vector products: each unordered tile pair once (the
// tiling, slots and conflict-free j side of k_rhs_sym_f32x2). For the pair
// (i, j), with d = x'_i - x'_j and the negated db' = beta_j - beta_i of
// k_hess_f32x2, s1 = p_j.a_i + p_i.a_j, p_i.p_j and d.db' are symmetric; the
// j terms follow from the i terms by d -> -d, db' -> -db':
//   i: Apq += t1 d,  App += g a_j,  Aqq += w z,  Aqp' += m p_j
//   j: Apq -= t1 d,  App += g a_i,  Aqq -= w z,  Aqp' += m p_i
// (t1 = g s1, w = g p_i.p_j, z = uu d + db', uu = -c1 d.db', m = g d.db'; Aqp'
// is stored negated as in k_hess_f32x2). Per unordered pair: 28 packed-pair
// FP32 ops shared + 2 x 12 accumulations = 52 FP32 + 1 MUFU (gather: 74 + 2).
template <int TPT, int NT, int MINB, int SB>
__global__ void __launch_bounds__(NT, MINB)
    k_hess_sym_f32x2(const float4* __restrict__ rec, const float4* __restrict__ adj, int n,
                     int T, float kap, float kc0x, float kc0y, float kc0z, float c1,
                     float4* __restrict__ part, int k0 = -1) {
  constexpr int TP = TPT / 2, TILE = NT * TPT, NW = NT / 32;
  static_assert(TILE % SB == 0 && SB % 32 == 0 && TPT % 2 == 0, "tile shape");
  __shared__ float4 sq[SB], sp[SB], sa[SB], sb[SB];
  __shared__ float4 sj[NW][3][SB];
  // k0 >= 0: diagonal group (slots 2(k - k0) / 2(k - k0) + 1), as k_rhs_sym_f32x2
  const int I = blockIdx.x, k = (k0 < 0 ? 0 : k0) + blockIdx.y;
  const int J = I + k < T ? I + k : I + k - T;
  const size_t slot_i = k0 < 0 ? (size_t)J : (size_t)(2 * (k - k0));
  const size_t slot_j = k0 < 0 ? (size_t)I : (size_t)(2 * (k - k0) + 1);
  if (2 * k == T && I >= k) {  // even T: the pair {I, I + T/2} once
    if (k0 >= 0) {
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int u = threadIdx.x; u < TILE; u += NT) {
        const int t = I * TILE + u, j = J * TILE + u;
        for (int c = 0; c < 4; ++c) {
          if (t < n) part[4 * (slot_i * n + t) + c] = z;
          if (j < n) part[4 * (slot_j * n + j) + c] = z;
        }
      }
    }
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  f2 qx[TP], qy[TP], qz[TP], px[TP], py[TP], pz[TP];
  f2 ix[TP], iy[TP], iz[TP], jx[TP], jy[TP], jz[TP];  // alpha_i, beta_i
  f2 A[TP][12];
  const int tb = I * TILE + threadIdx.x;
#pragma unroll
  for (int kk = 0; kk < TP; ++kk) {
    float4 q[2], p[2], al[2], be[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = tb + (2 * kk + h) * NT;
      q[h] = p[h] = al[h] = be[h] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < n) {
        q[h] = rec[2 * t]; p[h] = rec[2 * t + 1]; al[h] = adj[2 * t]; be[h] = adj[2 * t + 1];
      }
      q[h] = make_float4(fmaf(kap, q[h].x, -kc0x), fmaf(kap, q[h].y, -kc0y), fmaf(kap, q[h].z, -kc0z), 0.f);
    }
    qx[kk] = pk2(q[0].x, q[1].x); qy[kk] = pk2(q[0].y, q[1].y); qz[kk] = pk2(q[0].z, q[1].z);
    px[kk] = pk2(p[0].x, p[1].x); py[kk] = pk2(p[0].y, p[1].y); pz[kk] = pk2(p[0].z, p[1].z);
    ix[kk] = pk2(al[0].x, al[1].x); iy[kk] = pk2(al[0].y, al[1].y); iz[kk] = pk2(al[0].z, al[1].z);
    jx[kk] = pk2(be[0].x, be[1].x); jy[kk] = pk2(be[0].y, be[1].y); jz[kk] = pk2(be[0].z, be[1].z);
#pragma unroll
    for (int c = 0; c < 12; ++c) A[kk][c] = pk2(0.f, 0.f);
  }
  const f2 cc1 = bc2(-c1);
  const int jbase = J * TILE;
  for (int st = 0; st < TILE; st += SB) {
    __syncthreads();
    for (int u = threadIdx.x; u < SB; u += NT) {
      const int j = jbase + st + u;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f), p = q, a = q, b = q;
      if (j < n) {
        q = rec[2 * j]; p = rec[2 * j + 1]; a = adj[2 * j]; b = adj[2 * j + 1];
        q = make_float4(fmaf(kap, q.x, -kc0x), fmaf(kap, q.y, -kc0y), fmaf(kap, q.z, -kc0z), 0.f);
      }
      sq[u] = q; sp[u] = p; sa[u] = a; sb[u] = b;  // zero records contribute exactly 0
    }
    __syncthreads();
    for (int b0 = 0; b0 < SB; b0 += 32) {
     // j sums of source (lane + s) mod 32, travelling with it from lane to lane
     f2 Jv[12];
#pragma unroll
     for (int c = 0; c < 12; ++c) Jv[c] = pk2(0.f, 0.f);
     for (int s = 0; s < 32; ++s) {
      // diagonal pair: gather over every source; else lane l takes source
      // (l + s) mod 32 of the current 32-source batch
      const int u = b0 + (k == 0 ? s : ((lane + s) & 31));
      const float4 Q = sq[u], P = sp[u], Al = sa[u], Be = sb[u];
      const f2 Qx = bc2(Q.x), Qy = bc2(Q.y), Qz = bc2(Q.z);
      const f2 Px = bc2(P.x), Py = bc2(P.y), Pz = bc2(P.z);
      const f2 Ax = bc2(Al.x), Ay = bc2(Al.y), Az = bc2(Al.z);
      const f2 Bx = bc2(Be.x), By = bc2(Be.y), Bz = bc2(Be.z);
#pragma unroll
      for (int kk = 0; kk < TP; ++kk) {
        const f2 dx = sub2(qx[kk], Qx), dy = sub2(qy[kk], Qy), dz = sub2(qz[kk], Qz);
        f2 r2 = mul2(dx, dx);
        r2 = fma2(dy, dy, r2);
        r2 = fma2(dz, dz, r2);
        const f2 g = nex2x2(r2);
        const f2 dbx = sub2(Bx, jx[kk]), dby = sub2(By, jy[kk]), dbz = sub2(Bz, jz[kk]);
        f2 ddb = mul2(dx, dbx);
        ddb = fma2(dy, dby, ddb);
        ddb = fma2(dz, dbz, ddb);
        f2 s1 = mul2(ix[kk], Px);
        s1 = fma2(iy[kk], Py, s1);
        s1 = fma2(iz[kk], Pz, s1);
        s1 = fma2(px[kk], Ax, s1);
        s1 = fma2(py[kk], Ay, s1);
        s1 = fma2(pz[kk], Az, s1);
        f2 pp = mul2(px[kk], Px);
        pp = fma2(py[kk], Py, pp);
        pp = fma2(pz[kk], Pz, pp);
        const f2 t1 = mul2(g, s1);
        A[kk][0] = fma2(t1, dx, A[kk][0]); A[kk][1] = fma2(t1, dy, A[kk][1]); A[kk][2] = fma2(t1, dz, A[kk][2]);
        A[kk][3] = fma2(g, Ax, A[kk][3]); A[kk][4] = fma2(g, Ay, A[kk][4]); A[kk][5] = fma2(g, Az, A[kk][5]);
        const f2 w = mul2(g, pp);
        const f2 uu = mul2(ddb, cc1);  // cc1 = -c1
        const f2 zx = fma2(uu, dx, dbx), zy = fma2(uu, dy, dby), zz = fma2(uu, dz, dbz);
        A[kk][6] = fma2(w, zx, A[kk][6]); A[kk][7] = fma2(w, zy, A[kk][7]); A[kk][8] = fma2(w, zz, A[kk][8]);
        const f2 m = mul2(g, ddb);
        A[kk][9] = fma2(m, Px, A[kk][9]); A[kk][10] = fma2(m, Py, A[kk][10]); A[kk][11] = fma2(m, Pz, A[kk][11]);
        if (k == 0) continue;
        Jv[0] = fma2(t1, dx, Jv[0]); Jv[1] = fma2(t1, dy, Jv[1]); Jv[2] = fma2(t1, dz, Jv[2]);
        Jv[3] = fma2(g, ix[kk], Jv[3]); Jv[4] = fma2(g, iy[kk], Jv[4]); Jv[5] = fma2(g, iz[kk], Jv[5]);
        Jv[6] = fma2(w, zx, Jv[6]); Jv[7] = fma2(w, zy, Jv[7]); Jv[8] = fma2(w, zz, Jv[8]);
        Jv[9] = fma2(m, px[kk], Jv[9]); Jv[10] = fma2(m, py[kk], Jv[10]); Jv[11] = fma2(m, pz[kk], Jv[11]);
      }
      if (k == 0) continue;
      const int from = (lane + 1) & 31;
#pragma unroll
      for (int c = 0; c < 12; ++c) Jv[c].v = __shfl_sync(0xffffffffu, Jv[c].v, from);
     }
     if (k != 0) {  // lane l now holds source b0 + l's sums over the warp's targets
      float f[12];
#pragma unroll
      for (int c = 0; c < 12; ++c) {
        float lo, hi;
        up2(Jv[c], lo, hi);
        f[c] = lo + hi;
      }
      const int u = b0 + lane;
      sj[warp][0][u] = make_float4(f[0], f[1], f[2], f[3]);
      sj[warp][1][u] = make_float4(f[4], f[5], f[6], f[7]);
      sj[warp][2][u] = make_float4(f[8], f[9], f[10], f[11]);
     }
    }
    if (k == 0) continue;
    __syncthreads();
    // j side of this sub-tile's sources, warp copies in warp order, slot I
    for (int u = threadIdx.x; u < SB; u += NT) {
      const int j = jbase + st + u;
      if (j < n) {
        float4 s0 = sj[0][0][u], s1 = sj[0][1][u], s2 = sj[0][2][u];
#pragma unroll
        for (int w = 1; w < NW; ++w) {
          const float4 t0 = sj[w][0][u], t1 = sj[w][1][u], t2 = sj[w][2][u];
          s0.x += t0.x; s0.y += t0.y; s0.z += t0.z; s0.w += t0.w;
          s1.x += t1.x; s1.y += t1.y; s1.z += t1.z; s1.w += t1.w;
          s2.x += t2.x; s2.y += t2.y; s2.z += t2.z; s2.w += t2.w;
        }
        // (Apq, App, Aqq, Aqp') of j = (-J0..2, J3..5, -J6..8, -J9..11)
        float4* o = part + 4 * (slot_j * n + j);
        o[0] = make_float4(-s0.x, -s0.y, -s0.z, 0.f);
        o[1] = make_float4(s0.w, s1.x, s1.y, 0.f);
        o[2] = make_float4(-s1.z, -s1.w, -s2.x, 0.f);
        o[3] = make_float4(-s2.y, -s2.z, -s2.w, 0.f);
      }
    }
  }
  // i side: slot J (the diagonal pair: J = I)
#pragma unroll
  for (int kk = 0; kk < TP; ++kk) {
    float v[2][12];
#pragma unroll
    for (int c = 0; c < 12; ++c) up2(A[kk][c], v[0][c], v[1][c]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = tb + (2 * kk + h) * NT;
      if (t < n) {
        float4* o = part + 4 * (slot_i * n + t);
        if (k0 >= 0 && k == 0)  // grouped diagonal: its j slot is zero
          for (int c = 0; c < 4; ++c) part[4 * (slot_j * n + t) + c] = make_float4(0.f, 0.f, 0.f, 0.f);
        o[0] = make_float4(v[h][0], v[h][1], v[h][2], 0.f);
        o[1] = make_float4(v[h][3], v[h][4], v[h][5], 0.f);
        o[2] = make_float4(v[h][6], v[h][7], v[h][8], 0.f);
        o[3] = make_float4(-v[h][9], -v[h][10], -v[h][11], 0.f);
      }
    }
  }
}

// FP64: the reference's own expression exp(-|d|^2 * inv_two_s) in unscaled
// coordinates; libdevice exp (no SFU path exists for FP64).
template <int TPT, int NT>
__global__ void __launch_bounds__(NT) k_rhs_f64(const double4* __restrict__ rec, int n,
                                                int tgt_begin, int n_tgt, int chunk,
                                                double inv_two_s, double4* __restrict__ part) {
  __shared__ double4 sq[kTile / 2];
  __shared__ double4 sp[kTile / 2];
  __shared__ double stab[64];  // 2^(j/64) for exp_nonpos (published by the first tile barrier)
  if (threadIdx.x < 64) stab[threadIdx.x] = kExp2Tab64[threadIdx.x];
  constexpr int tile = kTile / 2;
  double qx[TPT], qy[TPT], qz[TPT], px[TPT], py[TPT], pz[TPT];
  double ax[TPT], ay[TPT], az[TPT], bx[TPT], by[TPT], bz[TPT];
  const int tb = blockIdx.x * NT * TPT + threadIdx.x;
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int t = tb + k * NT;
    double4 q = make_double4(0, 0, 0, 0), p = q;
    if (t < n_tgt) {
      q = ld4(rec + 2 * (tgt_begin + t));
      p = ld4(rec + 2 * (tgt_begin + t) + 1);
    }
    qx[k] = q.x; qy[k] = q.y; qz[k] = q.z;
    px[k] = p.x; py[k] = p.y; pz[k] = p.z;
    ax[k] = ay[k] = az[k] = bx[k] = by[k] = bz[k] = 0.0;
  }
  const int j0 = blockIdx.y * chunk;
  const int j1 = min(n, j0 + chunk);
  for (int jt = j0; jt < j1; jt += tile) {
    __syncthreads();
    for (int u = threadIdx.x; u < tile; u += NT) {
      const int j = jt + u;
      double4 q = make_double4(0, 0, 0, 0), p = q;
      if (j < j1) {
        q = ld4(rec + 2 * j);
        p = ld4(rec + 2 * j + 1);
      }
      sq[u] = q;  // zero records (p = 0) contribute exactly 0
      sp[u] = p;
    }
    __syncthreads();
#pragma unroll kF64Unr
    for (int u = 0; u < tile; ++u) {
      const double4 a = sq[u];
      const double4 b = sp[u];
#pragma unroll
      for (int k = 0; k < TPT; ++k) {
        const double dx = qx[k] - a.x, dy = qy[k] - a.y, dz = qz[k] - a.z;
        const double r2 = dx * dx + dy * dy + dz * dz;
        const double g = exp_nonpos(-r2 * inv_two_s, stab);
        const double pp = px[k] * b.x + py[k] * b.y + pz[k] * b.z;
        const double c = pp * g;
        ax[k] += g * b.x; ay[k] += g * b.y; az[k] += g * b.z;
        bx[k] += c * dx; by[k] += c * dy; bz[k] += c * dz;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int t = tb + k * NT;
    if (t < n_tgt) {
      double4* o = part + 2 * ((size_t)blockIdx.y * n_tgt + t);
      st4(o, make_double4(ax[k], ay[k], az[k], 0.0));
      st4(o + 1, make_double4(bx[k], by[k], bz[k], 0.0));
    }
  }
}

// Symmetric exact FP64 RHS: the tiling and conflict-free j side of
// k_rhs_sym_f32x2 in double precision with the reference's own expression
// exp(-|d|^2 inv_two_s) (gs_exp.cuh). FP64 partials are 64 B, so instead of a
// slot per tile the tile pairs are launched in groups of diagonals [k0, k1):
// CTA (I, k) writes the i side of {I, I+k} to slot 2(k-k0) of tile I and the j
// side to slot 2(k-k0)+1 of tile J; the diagonal (k = 0) and the skipped
// even-T duplicates write zeros to the slot they would not otherwise fill, so
// every target has exactly 2(k1-k0) slots per group, folded (k_fold_group)
// into a running sum in fixed order: deterministic, with a 2 x Kg x n x 64 B
// buffer whatever N.
template <int TPT, int NT, int MINB, int SB>
__global__ void __launch_bounds__(NT, MINB)
    k_rhs_sym_f64(const double4* __restrict__ rec, int n, int T, int k0, double inv_two_s,
                  double4* __restrict__ part) {
  constexpr int TILE = NT * TPT, NW = NT / 32;
  static_assert(TILE % SB == 0 && SB % 32 == 0, "tile shape");
  __shared__ double4 sq[SB];
  __shared__ double4 sp[SB];
  __shared__ double2 sj[NW][3][SB];
  __shared__ double stab[64];
  if (threadIdx.x < 64) stab[threadIdx.x] = kExp2Tab64[threadIdx.x];
  const int I = blockIdx.x, k = k0 + blockIdx.y;
  const int J = I + k < T ? I + k : I + k - T;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tb = I * TILE + threadIdx.x;
  const size_t si = (size_t)(2 * (k - k0)) * n, sjs = si + n;  // slot offsets
  if (2 * k == T && I >= k) {
    // even T: the pair {I, I + T/2} belongs to CTA (I - T/2, T/2); fill the
    // slots this CTA would have written with zeros
    const double4 z = make_double4(0, 0, 0, 0);
    for (int u = threadIdx.x; u < TILE; u += NT) {
      const int t = I * TILE + u, j = J * TILE + u;
      if (t < n) { st4(part + 2 * (si + t), z); st4(part + 2 * (si + t) + 1, z); }
      if (j < n) { st4(part + 2 * (sjs + j), z); st4(part + 2 * (sjs + j) + 1, z); }
    }
    return;
  }
  double qx[TPT], qy[TPT], qz[TPT], px[TPT], py[TPT], pz[TPT];
  double ax[TPT], ay[TPT], az[TPT], bx[TPT], by[TPT], bz[TPT];
#pragma unroll
  for (int kk = 0; kk < TPT; ++kk) {
    const int t = tb + kk * NT;
    double4 q = make_double4(0, 0, 0, 0), p = q;
    if (t < n) {
      q = ld4(rec + 2 * t);
      p = ld4(rec + 2 * t + 1);
    }
    qx[kk] = q.x; qy[kk] = q.y; qz[kk] = q.z;
    px[kk] = p.x; py[kk] = p.y; pz[kk] = p.z;
    ax[kk] = ay[kk] = az[kk] = bx[kk] = by[kk] = bz[kk] = 0.0;
  }
  const int jbase = J * TILE;
  for (int st = 0; st < TILE; st += SB) {
    __syncthreads();
    for (int u = threadIdx.x; u < SB; u += NT) {
      const int j = jbase + st + u;
      double4 q = make_double4(0, 0, 0, 0), p = q;
      if (j < n) {
        q = ld4(rec + 2 * j);
        p = ld4(rec + 2 * j + 1);
      }
      sq[u] = q;  // zero records (p = 0) contribute exactly 0
      sp[u] = p;
    }
    __syncthreads();
    for (int b0 = 0; b0 < SB; b0 += 32) {
     // j sums of source (lane + s) mod 32, travelling with it from lane to lane
     double jax = 0, jay = 0, jaz = 0, jbx = 0, jby = 0, jbz = 0;
#pragma unroll 2
     for (int s = 0; s < 32; ++s) {
      const int u = b0 + (k == 0 ? s : ((lane + s) & 31));
      const double4 a = sq[u];
      const double4 b = sp[u];
#pragma unroll
      for (int kk = 0; kk < TPT; ++kk) {
        const double dx = qx[kk] - a.x, dy = qy[kk] - a.y, dz = qz[kk] - a.z;
        const double r2 = dx * dx + dy * dy + dz * dz;
        const double g = exp_nonpos(-r2 * inv_two_s, stab);
        const double pp = px[kk] * b.x + py[kk] * b.y + pz[kk] * b.z;
        const double c = pp * g;
        ax[kk] += g * b.x; ay[kk] += g * b.y; az[kk] += g * b.z;
        bx[kk] += c * dx; by[kk] += c * dy; bz[kk] += c * dz;
        jax += g * px[kk]; jay += g * py[kk]; jaz += g * pz[kk];
        jbx += c * dx; jby += c * dy; jbz += c * dz;
      }
      if (k == 0) continue;
      const int from = (lane + 1) & 31;
      jax = __shfl_sync(0xffffffffu, jax, from); jay = __shfl_sync(0xffffffffu, jay, from);
      jaz = __shfl_sync(0xffffffffu, jaz, from); jbx = __shfl_sync(0xffffffffu, jbx, from);
      jby = __shfl_sync(0xffffffffu, jby, from); jbz = __shfl_sync(0xffffffffu, jbz, from);
     }
     if (k != 0) {  // lane l now holds source b0 + l's sums over the warp's targets
      const int u = b0 + lane;
      sj[warp][0][u] = make_double2(jax, jay);
      sj[warp][1][u] = make_double2(jaz, jbx);
      sj[warp][2][u] = make_double2(jby, jbz);
     }
    }
    if (k == 0) continue;
    __syncthreads();
    for (int u = threadIdx.x; u < SB; u += NT) {
      const int j = jbase + st + u;
      if (j < n) {
        double2 s0 = sj[0][0][u], s1 = sj[0][1][u], s2 = sj[0][2][u];
#pragma unroll
        for (int w = 1; w < NW; ++w) {
          const double2 t0 = sj[w][0][u], t1 = sj[w][1][u], t2 = sj[w][2][u];
          s0.x += t0.x; s0.y += t0.y; s1.x += t1.x; s1.y += t1.y; s2.x += t2.x; s2.y += t2.y;
        }
        st4(part + 2 * (sjs + j), make_double4(s0.x, s0.y, s1.x, 0.0));
        st4(part + 2 * (sjs + j) + 1, make_double4(-s1.y, -s2.x, -s2.y, 0.0));
      }
    }
  }
#pragma unroll
  for (int kk = 0; kk < TPT; ++kk) {
    const int t = tb + kk * NT;
    if (t < n) {
      st4(part + 2 * (si + t), make_double4(ax[kk], ay[kk], az[kk], 0.0));
      st4(part + 2 * (si + t) + 1, make_double4(bx[kk], by[kk], bz[kk], 0.0));
      if (k == 0) {  // the diagonal has no j side: its j slot is zero
        st4(part + 2 * (sjs + t), make_double4(0, 0, 0, 0));
        st4(part + 2 * (sjs + t) + 1, make_double4(0, 0, 0, 0));
      }
    }
  }
}

// acc[t] (+)= sum over the group's S slots of part[s][t], in slot order
__global__ void k_fold_group(const double4* __restrict__ part, int S, int n, int first,
                             double4* __restrict__ acc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double4 a = first ? make_double4(0, 0, 0, 0) : ld4(acc + 2 * t);
  double4 b = first ? make_double4(0, 0, 0, 0) : ld4(acc + 2 * t + 1);
  for (int s = 0; s < S; ++s) {
    const double4 x = ld4(part + 2 * ((size_t)s * n + t)), y = ld4(part + 2 * ((size_t)s * n + t) + 1);
    a.x += x.x; a.y += x.y; a.z += x.z;
    b.x += y.x; b.y += y.y; b.z += y.z;
  }
  st4(acc + 2 * t, a);
  st4(acc + 2 * t + 1, b);
}

// ----------------------------------------------------------------------------
// Hessian-vector products (kernel_exact.hpp:53-69), gather form over all j:
//   Apq = sum g (p_j.a_i + p_i.a_j) d'     Aqq = sum g (p_i.p_j) ((d'.db) C1 d' - db)
//   App = sum g a_j                         Aqp = sum g (d'.db) p_j
// with db = b_i - b_j; constants applied by the backward epilogue.
// Sources: state records (q, p) of step k + adjoint records (alpha, beta).
// 40 FP32 + 1 SFU per pair.
// ----------------------------------------------------------------------------
template <int TPT, int NT>
__global__ void __launch_bounds__(NT) k_hess_f32(const float4* __restrict__ rec,
                                                 const float4* __restrict__ adj, int n,
                                                 int tgt_begin, int n_tgt, int chunk, float kap,
                                                 float kc0x, float kc0y, float kc0z, float c1,
                                                 float4* __restrict__ part) {
  __shared__ float4 sq[kTile / 2], sp[kTile / 2], sa[kTile / 2], sb[kTile / 2];
  constexpr int tile = kTile / 2;
  float qx[TPT], qy[TPT], qz[TPT], px[TPT], py[TPT], pz[TPT];
  float ix[TPT], iy[TPT], iz[TPT], jx[TPT], jy[TPT], jz[TPT];  // alpha_i, beta_i
  float4 A0[TPT], A1[TPT], A2[TPT], A3[TPT];
  const int tb = blockIdx.x * NT * TPT + threadIdx.x;
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int t = tb + k * NT;
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f), p = q, a = q, b = q;
    if (t < n_tgt) {
      const int i = tgt_begin + t;
      q = rec[2 * i]; p = rec[2 * i + 1]; a = adj[2 * i]; b = adj[2 * i + 1];
    }
    qx[k] = fmaf(kap, q.x, -kc0x); qy[k] = fmaf(kap, q.y, -kc0y); qz[k] = fmaf(kap, q.z, -kc0z);
    px[k] = p.x; py[k] = p.y; pz[k] = p.z;
    ix[k] = a.x; iy[k] = a.y; iz[k] = a.z;
    jx[k] = b.x; jy[k] = b.y; jz[k] = b.z;
    A0[k] = A1[k] = A2[k] = A3[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int j0 = blockIdx.y * chunk;
  const int j1 = min(n, j0 + chunk);
  for (int jt = j0; jt < j1; jt += tile) {
    __syncthreads();
    for (int u = threadIdx.x; u < tile; u += NT) {
      const int j = jt + u;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f), p = q, a = q, b = q;
      if (j < j1) {
        q = rec[2 * j]; p = rec[2 * j + 1]; a = adj[2 * j]; b = adj[2 * j + 1];
        q = make_float4(fmaf(kap, q.x, -kc0x), fmaf(kap, q.y, -kc0y), fmaf(kap, q.z, -kc0z), 0.f);
      }
      sq[u] = q; sp[u] = p; sa[u] = a; sb[u] = b;  // zero records contribute exactly 0
    }
    __syncthreads();
#pragma unroll 1
    for (int u = 0; u < tile; ++u) {
      const float4 Q = sq[u], P = sp[u], Al = sa[u], Be = sb[u];
#pragma unroll
      for (int k = 0; k < TPT; ++k) {
        const float dx = qx[k] - Q.x, dy = qy[k] - Q.y, dz = qz[k] - Q.z;
        float nr2 = -dx * dx;
        nr2 = fmaf(-dy, dy, nr2);
        nr2 = fmaf(-dz, dz, nr2);
        const float g = ex2(nr2);
        const float dbx = jx[k] - Be.x, dby = jy[k] - Be.y, dbz = jz[k] - Be.z;
        float ddb = dx * dbx;
        ddb = fmaf(dy, dby, ddb);
        ddb = fmaf(dz, dbz, ddb);
        float s1 = P.x * ix[k];
        s1 = fmaf(P.y, iy[k], s1);
        s1 = fmaf(P.z, iz[k], s1);
        s1 = fmaf(px[k], Al.x, s1);
        s1 = fmaf(py[k], Al.y, s1);
        s1 = fmaf(pz[k], Al.z, s1);
        float pp = px[k] * P.x;
        pp = fmaf(py[k], P.y, pp);
        pp = fmaf(pz[k], P.z, pp);
        const float t1 = g * s1;
        A0[k].x = fmaf(t1, dx, A0[k].x); A0[k].y = fmaf(t1, dy, A0[k].y); A0[k].z = fmaf(t1, dz, A0[k].z);
        A1[k].x = fmaf(g, Al.x, A1[k].x); A1[k].y = fmaf(g, Al.y, A1[k].y); A1[k].z = fmaf(g, Al.z, A1[k].z);
        const float w = g * pp;
        const float uu = ddb * c1;
        const float zx = fmaf(uu, dx, -dbx), zy = fmaf(uu, dy, -dby), zz = fmaf(uu, dz, -dbz);
        A2[k].x = fmaf(w, zx, A2[k].x); A2[k].y = fmaf(w, zy, A2[k].y); A2[k].z = fmaf(w, zz, A2[k].z);
        const float m = g * ddb;
        A3[k].x = fmaf(m, P.x, A3[k].x); A3[k].y = fmaf(m, P.y, A3[k].y); A3[k].z = fmaf(m, P.z, A3[k].z);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int t = tb + k * NT;
    if (t < n_tgt) {
      float4* o = part + 4 * ((size_t)blockIdx.y * n_tgt + t);
      o[0] = A0[k]; o[1] = A1[k]; o[2] = A2[k]; o[3] = A3[k];
    }
  }
}

template <int TPT, int NT>
__global__ void __launch_bounds__(NT) k_hess_f64(const double4* __restrict__ rec,
                                                 const double4* __restrict__ adj, int n,
                                                 int tgt_begin, int n_tgt, int chunk,
                                                 double inv_two_s, double inv_s,
                                                 double4* __restrict__ part) {
  constexpr int tile = kTile / 4;
  __shared__ double4 sq[tile], sp[tile], sa[tile], sb[tile];
  __shared__ double stab[64];  // 2^(j/64) for exp_nonpos (published by the first tile barrier)
  if (threadIdx.x < 64) stab[threadIdx.x] = kExp2Tab64[threadIdx.x];
  double qx[TPT], qy[TPT], qz[TPT], px[TPT], py[TPT], pz[TPT];
  double ix[TPT], iy[TPT], iz[TPT], jx[TPT], jy[TPT], jz[TPT];
  double A[TPT][12];
  const int tb = blockIdx.x * NT * TPT + threadIdx.x;
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int t = tb + k * NT;
    double4 q = make_double4(0, 0, 0, 0), p = q, a = q, b = q;
    if (t < n_tgt) {
      const int i = tgt_begin + t;
      q = ld4(rec + 2 * i); p = ld4(rec + 2 * i + 1); a = ld4(adj + 2 * i); b = ld4(adj + 2 * i + 1);
    }
    qx[k] = q.x; qy[k] = q.y; qz[k] = q.z; px[k] = p.x; py[k] = p.y; pz[k] = p.z;
    ix[k] = a.x; iy[k] = a.y; iz[k] = a.z; jx[k] = b.x; jy[k] = b.y; jz[k] = b.z;
#pragma unroll
    for (int c = 0; c < 12; ++c) A[k][c] = 0.0;
  }
  const int j0 = blockIdx.y * chunk;
  const int j1 = min(n, j0 + chunk);
  for (int jt = j0; jt < j1; jt += tile) {
    __syncthreads();
    for (int u = threadIdx.x; u < tile; u += NT) {
      const int j = jt + u;
      double4 q = make_double4(0, 0, 0, 0), p = q, a = q, b = q;
      if (j < j1) {
        q = ld4(rec + 2 * j); p = ld4(rec + 2 * j + 1); a = ld4(adj + 2 * j); b = ld4(adj + 2 * j + 1);
      }
      sq[u] = q; sp[u] = p; sa[u] = a; sb[u] = b;
    }
    __syncthreads();
    for (int u = 0; u < tile; ++u) {
      const double4 Q = sq[u], P = sp[u], Al = sa[u], Be = sb[u];
#pragma unroll
      for (int k = 0; k < TPT; ++k) {
        const double dx = qx[k] - Q.x, dy = qy[k] - Q.y, dz = qz[k] - Q.z;
        const double g = exp_nonpos(-(dx * dx + dy * dy + dz * dz) * inv_two_s, stab);
        const double dbx = jx[k] - Be.x, dby = jy[k] - Be.y, dbz = jz[k] - Be.z;
        const double ddb = dx * dbx + dy * dby + dz * dbz;
        const double s1 = (P.x * ix[k] + P.y * iy[k] + P.z * iz[k]) +
                          (px[k] * Al.x + py[k] * Al.y + pz[k] * Al.z);
        const double pp = px[k] * P.x + py[k] * P.y + pz[k] * P.z;
        const double t1 = g * s1;
        A[k][0] += t1 * dx; A[k][1] += t1 * dy; A[k][2] += t1 * dz;
        A[k][3] += g * Al.x; A[k][4] += g * Al.y; A[k][5] += g * Al.z;
        const double w = g * pp, uu = ddb * inv_s;
        A[k][6] += w * (uu * dx - dbx); A[k][7] += w * (uu * dy - dby); A[k][8] += w * (uu * dz - dbz);
        const double m = g * ddb;
        A[k][9] += m * P.x; A[k][10] += m * P.y; A[k][11] += m * P.z;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int t = tb + k * NT;
    if (t < n_tgt) {
      double4* o = part + 4 * ((size_t)blockIdx.y * n_tgt + t);
      st4(o + 0, make_double4(A[k][0], A[k][1], A[k][2], 0.0));
      st4(o + 1, make_double4(A[k][3], A[k][4], A[k][5], 0.0));
      st4(o + 2, make_double4(A[k][6], A[k][7], A[k][8], 0.0));
      st4(o + 3, make_double4(A[k][9], A[k][10], A[k][11], 0.0));
    }
  }
}

// ----------------------------------------------------------------------------
// Velocity field v(x) = sum_j G(|x - q_j|) p_j at separate eval points
// (exact_velocity, kernel_exact.cpp:70-82; warp, shooting.cpp:288-294).
// 9 FP32 + 1 SFU per pair. Eval points: records of (x, unused).
// ----------------------------------------------------------------------------
// Packed variant of k_vel_f32 (exact_velocity / the dense warp): TPT
// evaluation points per thread as TPT/2 register pairs; per two (point,
// source) pairs 3 FADD2 + FMUL2 + 2 FFMA2 (-r^2) + 2 MUFU + 3 FFMA2 (sum g p)
// = 9 packed + 2 MUFU issue slots (scalar: 20): FMA-pipe bound at 9 FP32 per
// pair instead of issue bound at 10 instructions per pair.
template <int TPT, int NT>
__global__ void __launch_bounds__(NT) k_vel_f32x2(const float4* __restrict__ rec, int n,
                                                  const float4* __restrict__ ev, int m, int chunk,
                                                  float kap, float kc0x, float kc0y, float kc0z,
                                                  float4* __restrict__ part) {
  constexpr int TP = TPT / 2;
  __shared__ float4 sq[kTile], sp[kTile];
  f2 qx[TP], qy[TP], qz[TP], ax[TP], ay[TP], az[TP];
  const int tb = blockIdx.x * NT * TPT + threadIdx.x;
#pragma unroll
  for (int k = 0; k < TP; ++k) {
    float4 x[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = tb + (2 * k + h) * NT;
      x[h] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < m) x[h] = ev[2 * t];
      x[h] = make_float4(fmaf(kap, x[h].x, -kc0x), fmaf(kap, x[h].y, -kc0y), fmaf(kap, x[h].z, -kc0z), 0.f);
    }
    qx[k] = pk2(x[0].x, x[1].x); qy[k] = pk2(x[0].y, x[1].y); qz[k] = pk2(x[0].z, x[1].z);
    ax[k] = ay[k] = az[k] = pk2(0.f, 0.f);
  }
  const int j0 = blockIdx.y * chunk;
  const int j1 = min(n, j0 + chunk);
  for (int jt = j0; jt < j1; jt += kTile) {
    __syncthreads();
    for (int u = threadIdx.x; u < kTile; u += NT) {
      const int j = jt + u;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f), p = q;
      if (j < j1) {
        q = rec[2 * j]; p = rec[2 * j + 1];
        q = make_float4(fmaf(kap, q.x, -kc0x), fmaf(kap, q.y, -kc0y), fmaf(kap, q.z, -kc0z), 0.f);
      }
      sq[u] = q; sp[u] = p;  // zero records contribute exactly 0 (p = 0)
    }
    __syncthreads();
#pragma unroll 8
    for (int u = 0; u < kTile; ++u) {
      const float4 a = sq[u], b = sp[u];
      const f2 axx = bc2(a.x), ayy = bc2(a.y), azz = bc2(a.z);
      const f2 bxx = bc2(b.x), byy = bc2(b.y), bzz = bc2(b.z);
      f2 g[TP];
#pragma unroll
      for (int k = 0; k < TP; ++k) {
        const f2 dx = sub2(qx[k], axx), dy = sub2(qy[k], ayy), dz = sub2(qz[k], azz);
        f2 r2 = mul2(dx, dx);
        r2 = fma2(dy, dy, r2);
        r2 = fma2(dz, dz, r2);
        g[k] = nex2x2(r2);
      }
#pragma unroll
      for (int k = 0; k < TP; ++k) {
        ax[k] = fma2(g[k], bxx, ax[k]); ay[k] = fma2(g[k], byy, ay[k]); az[k] = fma2(g[k], bzz, az[k]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < TP; ++k) {
    float lx[2], ly[2], lz[2];
    up2(ax[k], lx[0], lx[1]); up2(ay[k], ly[0], ly[1]); up2(az[k], lz[0], lz[1]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = tb + (2 * k + h) * NT;
      if (t < m) part[(size_t)blockIdx.y * m + t] = make_float4(lx[h], ly[h], lz[h], 0.f);
    }
  }
}

template <int TPT, int NT>
__global__ void __launch_bounds__(NT) k_vel_f32(const float4* __restrict__ rec, int n,
                                                const float4* __restrict__ ev, int m, int chunk,
                                                float kap, float kc0x, float kc0y, float kc0z,
                                                float4* __restrict__ part) {
  __shared__ float4 sq[kTile], sp[kTile];
  float qx[TPT], qy[TPT], qz[TPT], ax[TPT], ay[TPT], az[TPT];
  const int tb = blockIdx.x * NT * TPT + threadIdx.x;
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int t = tb + k * NT;
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (t < m) x = ev[2 * t];
    qx[k] = fmaf(kap, x.x, -kc0x); qy[k] = fmaf(kap, x.y, -kc0y); qz[k] = fmaf(kap, x.z, -kc0z);
    ax[k] = ay[k] = az[k] = 0.f;
  }
  const int j0 = blockIdx.y * chunk;
  const int j1 = min(n, j0 + chunk);
  for (int jt = j0; jt < j1; jt += kTile) {
    __syncthreads();
    for (int u = threadIdx.x; u < kTile; u += NT) {
      const int j = jt + u;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f), p = q;
      if (j < j1) {
        q = rec[2 * j]; p = rec[2 * j + 1];
        q = make_float4(fmaf(kap, q.x, -kc0x), fmaf(kap, q.y, -kc0y), fmaf(kap, q.z, -kc0z), 0.f);
      }
      sq[u] = q; sp[u] = p;
    }
    __syncthreads();
#pragma unroll 2
    for (int u = 0; u < kTile; ++u) {
      const float4 a = sq[u], b = sp[u];
#pragma unroll
      for (int k = 0; k < TPT; ++k) {
        const float dx = qx[k] - a.x, dy = qy[k] - a.y, dz = qz[k] - a.z;
        float nr2 = -dx * dx;
        nr2 = fmaf(-dy, dy, nr2);
        nr2 = fmaf(-dz, dz, nr2);
        const float g = ex2(nr2);
        ax[k] = fmaf(g, b.x, ax[k]); ay[k] = fmaf(g, b.y, ay[k]); az[k] = fmaf(g, b.z, az[k]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int t = tb + k * NT;
    if (t < m) part[(size_t)blockIdx.y * m + t] = make_float4(ax[k], ay[k], az[k], 0.f);
  }
}

template <int TPT, int NT>
__global__ void __launch_bounds__(NT) k_vel_f64(const double4* __restrict__ rec, int n,
                                                const double4* __restrict__ ev, int m, int chunk,
                                                double inv_two_s, double4* __restrict__ part) {
  constexpr int tile = kTile / 2;
  __shared__ double4 sq[tile], sp[tile];
  __shared__ double stab[64];  // 2^(j/64) for exp_nonpos (published by the first tile barrier)
  if (threadIdx.x < 64) stab[threadIdx.x] = kExp2Tab64[threadIdx.x];
  double qx[TPT], qy[TPT], qz[TPT], ax[TPT], ay[TPT], az[TPT];
  const int tb = blockIdx.x * NT * TPT + threadIdx.x;
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int t = tb + k * NT;
    double4 x = make_double4(0, 0, 0, 0);
    if (t < m) x = ld4(ev + 2 * t);
    qx[k] = x.x; qy[k] = x.y; qz[k] = x.z;
    ax[k] = ay[k] = az[k] = 0.0;
  }
  const int j0 = blockIdx.y * chunk;
  const int j1 = min(n, j0 + chunk);
  for (int jt = j0; jt < j1; jt += tile) {
    __syncthreads();
    for (int u = threadIdx.x; u < tile; u += NT) {
      const int j = jt + u;
      double4 q = make_double4(0, 0, 0, 0), p = q;
      if (j < j1) { q = ld4(rec + 2 * j); p = ld4(rec + 2 * j + 1); }
      sq[u] = q; sp[u] = p;
    }
    __syncthreads();
    for (int u = 0; u < tile; ++u) {
      const double4 a = sq[u], b = sp[u];
#pragma unroll
      for (int k = 0; k < TPT; ++k) {
        const double dx = qx[k] - a.x, dy = qy[k] - a.y, dz = qz[k] - a.z;
        const double g = exp_nonpos(-(dx * dx + dy * dy + dz * dz) * inv_two_s, stab);
        ax[k] += g * b.x; ay[k] += g * b.y; az[k] += g * b.z;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int t = tb + k * NT;
    if (t < m) st4(part + (size_t)blockIdx.y * m + t, make_double4(ax[k], ay[k], az[k], 0.0));
  }
}

// ----------------------------------------------------------------------------
// launch planning
// ----------------------------------------------------------------------------
namespace {

struct Plan {
  int tpt, S, chunk;
  dim3 grid;
};

// Choose targets-per-thread and the number of source chunks S so that the
// grid covers an integral number of waves of resident CTAs.
Plan plan(int n_src, int n_tgt, int nt, const int* tpts, int ntpt, int tile, int occ,
          int sms) {
  const long slots = (long)occ * sms;
  Plan pl{};
  int tpt = tpts[ntpt - 1];
  for (int i = 0; i < ntpt; ++i) {
    const long b = (n_tgt + (long)nt * tpts[i] - 1) / ((long)nt * tpts[i]);
    if (b * 16 >= 2 * slots) { tpt = tpts[i]; break; }
  }
  const long B = (n_tgt + (long)nt * tpt - 1) / ((long)nt * tpt);
  const int smax = (int)std::max(1L, std::min((long)kMaxChunks, ((long)n_src + tile - 1) / tile));
  // S is chosen for the whole problem AND its 2/4/8-way target shards (those
  // that can fill a wave at all): score = worst wave efficiency over them +
  // half the unsharded one. Multi-device shards launch under this same plan
  // (rhs_partials plan_tgt), so one S -- hence bit-identical per-target sums --
  // serves every device count while each shard's grid still fills its GPU
  // (N = 1M, TPT 12: S = 14, 99.5 % of the last wave used unsharded, >= 96 %
  // for 2-8 shards).
  int bestS = 1;
  double best = -1.0;
  for (int s = 1; s <= smax; ++s) {
    double worst = 2.0;
    for (int g = 1; g <= 8; g *= 2) {
      const long Bg = (B + g - 1) / g;
      if (g > 1 && Bg * smax < slots) continue;  // this shard cannot fill a wave anyway
      const double w = (double)(Bg * s) / slots;
      worst = std::min(worst, w / std::ceil(w));
    }
    const double w1 = (double)(B * s) / slots;
    const double score = worst + 0.5 * (w1 / std::ceil(w1));
    // prefer fewer chunks unless clearly better balanced
    if (score > best + 0.01) { best = score; bestS = s; }
  }
  pl.tpt = tpt;
  pl.S = bestS;
  pl.chunk = (int)(((long)n_src + bestS - 1) / bestS);
  pl.chunk = (pl.chunk + tile - 1) / tile * tile;
  pl.S = (int)(((long)n_src + pl.chunk - 1) / pl.chunk);
  if (pl.S < 1) pl.S = 1;
  pl.grid = dim3((unsigned)B, (unsigned)pl.S, 1);
  return pl;
}

template <typename K>
int occupancy(K kernel, int nt) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, nt, 0);
  return occ > 0 ? occ : 1;
}

}  // namespace

constexpr int kNT = 128;

// Dispatch helpers: one instantiation per TPT.
#define GS_TPT_SWITCH(tpt, KERNEL, ...)                                   \
  switch (tpt) {                                                          \
    case 8: KERNEL<8, kNT><<<pl.grid, kNT, 0, st>>>(__VA_ARGS__); break;  \
    case 4: KERNEL<4, kNT><<<pl.grid, kNT, 0, st>>>(__VA_ARGS__); break;  \
    case 2: KERNEL<2, kNT><<<pl.grid, kNT, 0, st>>>(__VA_ARGS__); break;  \
    default: KERNEL<1, kNT><<<pl.grid, kNT, 0, st>>>(__VA_ARGS__); break; \
  }

// Gather FP32 RHS variants (shards and problems below 40k points), chosen by
// size: 0 = packed TPT 8 (3 CTAs/SM), 1 = packed TPT 12 from 500k targets,
// 2 = packed TPT 2 for grids that would not fill the GPU, 3 = scalar TPT 1
// for tiny problems; all with the source loop unrolled 8. GS_RHS_VARIANT
// forces one (the small-grid fallbacks still apply). Round 1 also measured
// scalar TPT 4 / 6 / 8, unphased, 4-CTA, TPT 16 and 4x-unrolled variants
// (profiles/r01_sweep_rhs_*.jsonl); they were slower and are no longer built.
struct RhsVariant {
  int tpt, minb;
};
static const RhsVariant kRhsVariants[] = {{8, 3}, {12, 2}, {2, 8}, {1, 8}};
constexpr int kNumRhsVariants = sizeof(kRhsVariants) / sizeof(kRhsVariants[0]);

static int rhs_variant() {
  static int v = [] {
    const char* e = std::getenv("GS_RHS_VARIANT");
    const int x = e ? std::atoi(e) : -1;
    return (x >= 0 && x < kNumRhsVariants) ? x : -1;
  }();
  return v;
}

template <int TPT, int MINB>
static void launch_rhs_f32(const Plan& pl, cudaStream_t st, const float4* rec, int n, int tb,
                           int nt, const KernelConsts& kc, float4* part) {
  k_rhs_f32<TPT, kNT, MINB><<<pl.grid, kNT, 0, st>>>(
      rec, n, tb, nt, pl.chunk, (float)kc.kappa, (float)(kc.kappa * kc.c0[0]),
      (float)(kc.kappa * kc.c0[1]), (float)(kc.kappa * kc.c0[2]), part);
}

template <int TPT, int MINB>
static int occ_rhs_f32() {
  return occupancy(k_rhs_f32<TPT, kNT, MINB>, kNT);
}

template <int TPT, int MINB, int UNR = 2>
static void launch_rhs_f32x2(const Plan& pl, cudaStream_t st, const float4* rec, int n, int tb,
                             int nt, const KernelConsts& kc, float4* part) {
  k_rhs_f32x2<TPT, kNT, MINB, UNR><<<pl.grid, kNT, 0, st>>>(
      rec, n, tb, nt, pl.chunk, (float)kc.kappa, (float)(kc.kappa * kc.c0[0]),
      (float)(kc.kappa * kc.c0[1]), (float)(kc.kappa * kc.c0[2]), part);
}

template <int TPT, int MINB, int UNR = 2>
static int occ_rhs_f32x2() {
  return occupancy(k_rhs_f32x2<TPT, kNT, MINB, UNR>, kNT);
}

// Exact FP32 RHS over Morton-ordered points (morton_order) with the
// underflow cutoff cut2 (scaled units; +inf: no tile skipped). Returns S.
int rhs_sorted_partials(const Device& dev, const void* srec, const int* perm, int n,
                        void* part, int part_cap_chunks, DBuf& boxes, float cut2,
                        cudaStream_t st) {
  // one warp per CTA: the CTA's 256 targets are one Morton group, so a tile is
  // skipped (load and compute) at the granularity of the group boxes
  constexpr int TPT = 8, NT = 32, MINB = 12;
  const int tgt_group = NT * TPT;
  const int nbt = (n + tgt_group - 1) / tgt_group, nbs = (n + kTile - 1) / kTile;
  GS_TRY_INT(boxes.ensure(sizeof(float4) * 2 * (size_t)(nbt + nbs)));
  float4* tbox = boxes.as<float4>();
  float4* sbox = tbox + 2 * nbt;
  k_group_boxes<<<nbt, 256, 0, st>>>((const float4*)srec, n, tgt_group, tbox);
  k_group_boxes<<<nbs, 256, 0, st>>>((const float4*)srec, n, kTile, sbox);
  static int occ = occupancy(k_rhs_f32x2_sorted<TPT, NT, MINB>, NT);
  const int tp[] = {TPT};
  Plan pl = plan(n, n, NT, tp, 1, kTile, occ, dev.sms);
  if (pl.S > part_cap_chunks) return -1;
  static const bool dbg = std::getenv("GS_EXACT_CUT_DEBUG") != nullptr;
  static unsigned long long* cnt = nullptr;
  if (dbg && !cnt) cudaMalloc(&cnt, 8);
  if (dbg) cudaMemsetAsync(cnt, 0, 8, st);
  k_rhs_f32x2_sorted<TPT, NT, MINB><<<pl.grid, NT, 0, st>>>(
      (const float4*)srec, perm, n, pl.chunk, tbox, sbox, cut2, (float4*)part, dbg ? cnt : nullptr);
  if (cudaGetLastError() != cudaSuccess) return -1;
  if (dbg) {
    unsigned long long h = 0;
    cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const double all = (double)((n + 255) / 256) * ((n + 255) / 256);
    std::fprintf(stderr, "[exact cut] S %d computed warp-tile pairs %llu of %.0f (%.2f %%)\n", pl.S, h,
                 all, 100.0 * h / all);
  }
  return pl.S;
}

// Grid of n_tgt targets under a plan made for plan_tgt targets: the kernel
// variant, targets per thread, source chunk count S and chunk length are those
// of the plan_tgt problem (so every target's partial sums are bit-identical to
// that problem's), only the target blocks are resized.
static Plan fit(Plan pl, int n_tgt) {
  pl.grid.x = (unsigned)std::max(1L, ((long)n_tgt + (long)kNT * pl.tpt - 1) / ((long)kNT * pl.tpt));
  return pl;
}

int rhs_partials(const Device& dev, int prec, const void* rec, int n, int tgt_begin, int n_tgt,
                 const KernelConsts& kc, void* part, int part_cap_chunks, cudaStream_t st,
                 int plan_tgt) {
  const int real_tgt = n_tgt;
  if (plan_tgt > 0) n_tgt = plan_tgt;  // plan as if for plan_tgt targets (multi-device shards)
  if (prec == kF32) {
    const int vi = rhs_variant();
    const long slots = 3L * dev.sms;
    // default: TPT 12 once the grid holds many waves of its larger blocks
    // (measured: 1.933 vs 1.913 Tpair/s at 1M; 1.81 vs 1.89 at 100k)
    int use = vi >= 0 ? vi : (n_tgt >= 500000 ? 1 : 0);
    // small problems: narrower target blocks so the grid fills the GPU
    const int tpt = kRhsVariants[use].tpt;
    if ((long)((n_tgt + kNT * tpt - 1) / (kNT * tpt)) * 16 < 2 * slots && use < 2) use = 2;
    if ((long)((n_tgt + kNT * 2 - 1) / (kNT * 2)) * 16 < 2 * slots) use = 3;
    const RhsVariant u = kRhsVariants[use];
    static int occs[kNumRhsVariants] = {occ_rhs_f32x2<8, 3, 8>(), occ_rhs_f32x2<12, 2, 8>(),
                                        occ_rhs_f32x2<2, 8, 8>(), occ_rhs_f32<1, 8>()};
    const int tp[] = {u.tpt};
    Plan pl = fit(plan(n, n_tgt, kNT, tp, 1, kTile, occs[use], dev.sms), real_tgt);
    if (pl.S > part_cap_chunks) return -1;
    const float4* r = (const float4*)rec;
    float4* o = (float4*)part;
    n_tgt = real_tgt;
    switch (use) {
      case 0: launch_rhs_f32x2<8, 3, 8>(pl, st, r, n, tgt_begin, n_tgt, kc, o); break;
      case 1: launch_rhs_f32x2<12, 2, 8>(pl, st, r, n, tgt_begin, n_tgt, kc, o); break;
      case 2: launch_rhs_f32x2<2, 8, 8>(pl, st, r, n, tgt_begin, n_tgt, kc, o); break;
      default: launch_rhs_f32<1, 8>(pl, st, r, n, tgt_begin, n_tgt, kc, o); break;
    }
    return pl.S;
  }
  static const int tpts[] = {4, 2, 1};
  static int occ = occupancy(k_rhs_f64<4, kNT>, kNT);
  Plan pl = fit(plan(n, n_tgt, kNT, tpts, 3, kTile / 2, occ, dev.sms), real_tgt);
  if (pl.S > part_cap_chunks) return -1;
  n_tgt = real_tgt;
  switch (pl.tpt) {
    case 4: k_rhs_f64<4, kNT><<<pl.grid, kNT, 0, st>>>((const double4*)rec, n, tgt_begin, n_tgt, pl.chunk, kc.inv_two_s, (double4*)part); break;
    case 2: k_rhs_f64<2, kNT><<<pl.grid, kNT, 0, st>>>((const double4*)rec, n, tgt_begin, n_tgt, pl.chunk, kc.inv_two_s, (double4*)part); break;
    default: k_rhs_f64<1, kNT><<<pl.grid, kNT, 0, st>>>((const double4*)rec, n, tgt_begin, n_tgt, pl.chunk, kc.inv_two_s, (double4*)part); break;
  }
  return pl.S;
}

// ---- symmetric exact FP32 RHS (k_rhs_sym_f32x2) -----------------------------
// gs_set_exact_pairs: 0 = by size (symmetric for large unsharded problems),
// 1 = gather (k_rhs_f32x2) always, 2 = symmetric whenever it applies.
static int g_exact_pairs = -1;
void set_exact_pairs(int mode) { g_exact_pairs = mode; }

static int exact_pairs_mode() {
  if (g_exact_pairs >= 0) return g_exact_pairs;
  static int m = [] {
    const char* e = std::getenv("GS_EXACT_PAIRS");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}

// Tile shapes, by size (tools/check_sym.py sweeps, profiles/r02_sym/): 0 =
// 12 targets x 256 threads (3072-point tiles, one CTA per SM) from 150k
// points; 1 = 12 x 128 (1536, two CTAs per SM) from 75k; 2 = 6 x 128 (768,
// three per SM) from 35k; 3 = 4 x 128 (512, four per SM) from 8k -- smaller
// tiles give the small problems enough tile pairs to fill the GPU (20k:
// 1.24x the gather kernel with 512-point tiles, 0.88x with 1536). Below 8k
// the gather kernel wins. Measured alternatives at 1M: 8 x
// 128 / 8 x 256 / 8 x 384 / 10 x 256 / 14 x 128 targets, 64- or 256-source
// sub-tiles, step unroll 2 / 4 / 16, the j side accumulated after the whole i
// side: all equal or slower.
struct SymShape {
  int tpt, nt;
};
static const SymShape kSym[] = {{12, 256}, {12, 128}, {6, 128}, {4, 128}};

static int sym_variant(int n) {
  static int forced = [] {
    const char* e = std::getenv("GS_SYM_VARIANT");
    return e ? std::atoi(e) : -1;
  }();
  if (forced >= 0 && forced <= 3) return forced;
  return n >= 150000 ? 0 : n >= 75000 ? 1 : n >= 35000 ? 2 : 3;
}

int sym_tiles(int n) {
  const SymShape s = kSym[sym_variant(n)];
  return (int)(((long)n + (long)s.tpt * s.nt - 1) / ((long)s.tpt * s.nt));
}

bool use_sym(int prec, int n, int tgt_begin, int n_tgt, int plan_tgt) {
  if (prec != kF32 || tgt_begin != 0 || n_tgt != n || plan_tgt > 0) return false;
  const int mode = exact_pairs_mode();
  if (mode == 1) return false;
  // (problems whose T slots x n x 32 B exceed kSymSlotBudget run in
  // diagonal groups folded into a running sum: rhs_sym_partials)
  if (mode == 2) return true;
  // by size: enough tile pairs to fill the GPU (T(T+1)/2 CTAs)
  return n >= 8000;
}

// One slot per tile up to kSymSlotBudget bytes of partials (1M points: 10.4
// GB); above it (from ~1.5M points) the diagonals run in groups of
// kSymGroup, each folded into a running sum (2 x kSymGroup slots + the sum).
constexpr double kSymSlotBudget = 24e9;
constexpr int kSymGroup = 32;

static double sym_slot_budget() {
  static const double budget = [] {  // GS_SYM_SLOT_BUDGET: test hook (bytes)
    const char* e = std::getenv("GS_SYM_SLOT_BUDGET");
    return e ? std::atof(e) : kSymSlotBudget;
  }();
  return budget;
}

bool sym_grouped(int n) { return (double)sym_tiles(n) * n * 32.0 > sym_slot_budget(); }

size_t sym_part_bytes(int n) {
  const size_t slots = sym_grouped(n) ? 1 + 2 * kSymGroup : sym_tiles(n);
  return slots * (size_t)n * 2 * sizeof(float4);
}

int sym_launches(int n) {
  return sym_grouped(n) ? 2 * ((sym_tiles(n) / 2 + 1 + kSymGroup - 1) / kSymGroup) : 1;
}

// k_rhs_sym_f32x2 in tile shape v (kSym) over grid (rows, diagonals)
static void launch_sym(int v, dim3 grid, cudaStream_t st, const float4* r, int n, int T,
                       float kap, float a, float b, float c, float4* o, int row0, int k0) {
  switch (v) {
    case 0: k_rhs_sym_f32x2<12, 256, 1, 128, 8><<<grid, 256, 0, st>>>(r, n, T, kap, a, b, c, o, row0, k0); break;
    case 1: k_rhs_sym_f32x2<12, 128, 2, 256, 4><<<grid, 128, 0, st>>>(r, n, T, kap, a, b, c, o, row0, k0); break;
    case 2: k_rhs_sym_f32x2<6, 128, 3, 128, 8><<<grid, 128, 0, st>>>(r, n, T, kap, a, b, c, o, row0, k0); break;
    default: k_rhs_sym_f32x2<4, 128, 4, 128, 8><<<grid, 128, 0, st>>>(r, n, T, kap, a, b, c, o, row0, k0); break;
  }
}

// Multi-GPU symmetric RHS: rank r of G evaluates the tile-pair
// rows I in [T r / G, T (r+1) / G) -- every unordered tile pair belongs to
// exactly one row, and rows are equally loaded (T/2 + 1 pairs each) -- and
// folds, for EVERY target, the slots its rows wrote (in slot order) into one
// partial (A, B). The ranks then exchange the partials of each target shard
// (all-to-all) and the shard's epilogue folds the G partials in rank order.
// owner(X, Y): the row whose CTA evaluates the pair {X, Y} (k = (Y - X) mod T;
// k <= T/2 -> X, except the even-T k = T/2 pairs, taken by min(X, Y); else Y).
__device__ __forceinline__ int pair_owner(int X, int Y, int T) {
  const int k = Y >= X ? Y - X : Y - X + T;
  if (2 * k == T) return min(X, Y);
  return 2 * k < T ? X : Y;
}

__global__ void k_fold_rows(const float4* __restrict__ part, int n, int T, int tile, int ra,
                            int rb, float4* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int X = t / tile;
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
  for (int Y = 0; Y < T; ++Y) {
    const int o = pair_owner(X, Y, T);
    if (o < ra || o >= rb) continue;
    const float4 u = part[2 * ((size_t)Y * n + t)], v = part[2 * ((size_t)Y * n + t) + 1];
    a.x += u.x; a.y += u.y; a.z += u.z;
    b.x += v.x; b.y += v.y; b.z += v.z;
  }
  out[2 * t] = a;
  out[2 * t + 1] = b;
}

int rhs_sym_rows(const void* rec, int n, const KernelConsts& kc, void* part, void* out, int rank,
                 int world, cudaStream_t st) {
  const int T = sym_tiles(n);
  const int v = sym_variant(n);
  const int tile = kSym[v].tpt * kSym[v].nt;
  const int ra = (int)((long)T * rank / world), rb = (int)((long)T * (rank + 1) / world);
  const float kap = (float)kc.kappa, a = (float)(kc.kappa * kc.c0[0]),
              b = (float)(kc.kappa * kc.c0[1]), c = (float)(kc.kappa * kc.c0[2]);
  const float4* r = (const float4*)rec;
  float4* o = (float4*)part;
  if (rb > ra) launch_sym(v, dim3((unsigned)(rb - ra), (unsigned)(T / 2 + 1), 1), st, r, n, T, kap, a, b, c, o, ra, -1);
  k_fold_rows<<<(n + 255) / 256, 256, 0, st>>>(o, n, T, tile, ra, rb, (float4*)out);
  return T;
}

int rhs_sym_partials(const void* rec, int n, const KernelConsts& kc, void* part, cudaStream_t st) {
  const int T = sym_tiles(n);
  const float kap = (float)kc.kappa, a = (float)(kc.kappa * kc.c0[0]),
              b = (float)(kc.kappa * kc.c0[1]), c = (float)(kc.kappa * kc.c0[2]);
  const float4* r = (const float4*)rec;
  const int v = sym_variant(n);
  if (!sym_grouped(n)) {
    launch_sym(v, dim3((unsigned)T, (unsigned)(T / 2 + 1), 1), st, r, n, T, kap, a, b, c,
               (float4*)part, 0, -1);
    return T;
  }
  float4* acc = (float4*)part;
  float4* slots = acc + 2 * (size_t)n;
  const int kend = T / 2 + 1;
  for (int k0 = 0; k0 < kend; k0 += kSymGroup) {
    const int k1 = std::min(kend, k0 + kSymGroup);
    launch_sym(v, dim3((unsigned)T, (unsigned)(k1 - k0), 1), st, r, n, T, kap, a, b, c, slots, 0, k0);
    k_fold_group_f32<<<(n + 255) / 256, 256, 0, st>>>(slots, 2 * (k1 - k0), n, k0 == 0, acc);
  }
  return 1;  // the epilogue reads the running sum as a single partial
}

#ifndef SYM_F64_BIG_N
#define SYM_F64_BIG_N 100000
#endif
#ifndef SYM_F64_MIN_N
#define SYM_F64_MIN_N 8000
#endif
// Symmetric FP64 RHS (k_rhs_sym_f64): 1024-point tiles (4 targets x 256
// threads), diagonal groups of kSymF64Group folded into a running sum.
// (512-point tiles -- 4 targets x 128 threads, two CTAs per SM -- below
// 100k points: enough tile pairs for the small problems)
constexpr int kSymF64Tile = 4 * 256, kSymF64TileSmall = 4 * 128, kSymF64Group = 32;
static int sym_f64_tile(int n) {
  static const int forced = [] {  // GS_SYM_F64_TILE: 1024 / 512 (sweeps)
    const char* e = std::getenv("GS_SYM_F64_TILE");
    return e ? std::atoi(e) : 0;
  }();
  if (forced == kSymF64Tile || forced == kSymF64TileSmall) return forced;
  return n >= SYM_F64_BIG_N ? kSymF64Tile : kSymF64TileSmall;
}
int sym_f64_tiles(int n) { return (n + sym_f64_tile(n) - 1) / sym_f64_tile(n); }

bool use_sym_f64(int n, int tgt_begin, int n_tgt, int plan_tgt) {
  if (tgt_begin != 0 || n_tgt != n || plan_tgt > 0) return false;
  const int mode = exact_pairs_mode();
  if (mode == 1) return false;
  return mode == 2 || n >= SYM_F64_MIN_N;
}

size_t sym_f64_part_bytes(int n) {
  // running sum (n x 64 B) + one group's slots (2 x group x n x 64 B)
  return (size_t)(1 + 2 * kSymF64Group) * (size_t)n * 2 * sizeof(double4);
}

int rhs_sym_f64_partials(const void* rec, int n, const KernelConsts& kc, void* part,
                         cudaStream_t st) {
  const int T = sym_f64_tiles(n);
  double4* acc = (double4*)part;
  double4* slots = acc + 2 * (size_t)n;
  const int kend = T / 2 + 1;
  for (int k0 = 0; k0 < kend; k0 += kSymF64Group) {
    const int k1 = std::min(kend, k0 + kSymF64Group);
    if (sym_f64_tile(n) == kSymF64TileSmall)
      k_rhs_sym_f64<4, 128, 2, 64><<<dim3((unsigned)T, (unsigned)(k1 - k0)), 128, 0, st>>>(
          (const double4*)rec, n, T, k0, kc.inv_two_s, slots);
    else
    k_rhs_sym_f64<4, 256, 1, 64><<<dim3((unsigned)T, (unsigned)(k1 - k0)), 256, 0, st>>>(
        (const double4*)rec, n, T, k0, kc.inv_two_s, slots);
    k_fold_group<<<(n + 255) / 256, 256, 0, st>>>(slots, 2 * (k1 - k0), n, k0 == 0, acc);
  }
  return 1;  // the epilogue reads the running sum as a single partial
}

int sym_f64_launches(int n) { return 2 * ((sym_f64_tiles(n) / 2 + 1 + kSymF64Group - 1) / kSymF64Group); }

#ifndef HESS_SYM_MIN_N
#define HESS_SYM_MIN_N 8000
#endif
// Symmetric Hessian products (k_hess_sym_f32x2): 768-point tiles (6 targets
// x 128 threads, two CTAs per SM), the same choice rules as the RHS.
// (512-point tiles -- 4 targets x 128 threads, three CTAs per SM -- below 40k
// points, so that small problems still fill the GPU with tile pairs)
constexpr int kHessSymTile = 6 * 128, kHessSymTileSmall = 4 * 128;
static int hess_sym_forced() {
  static const int v = [] {  // GS_HESS_SYM_TILE: 768 / 512 (sweeps)
    const char* e = std::getenv("GS_HESS_SYM_TILE");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}
static int hess_sym_tile(int n) {
  const int f = hess_sym_forced();
  if (f == kHessSymTile || f == kHessSymTileSmall) return f;
  return n >= 40000 ? kHessSymTile : kHessSymTileSmall;
}
static int hess_sym_tiles(int n) { return (n + hess_sym_tile(n) - 1) / hess_sym_tile(n); }

static bool use_sym_hess(int prec, int n, int tgt_begin, int n_tgt, int plan_tgt) {
  if (prec != kF32 || tgt_begin != 0 || n_tgt != n || plan_tgt > 0) return false;
  const int mode = exact_pairs_mode();
  if (mode == 1) return false;
  return mode == 2 || n >= HESS_SYM_MIN_N;
}

// slots over the budget: diagonal groups folded into a running sum (as the RHS)
static bool hess_sym_grouped(int n) { return (double)hess_sym_tiles(n) * n * 64.0 > sym_slot_budget(); }
constexpr int kHessSymGroup = 16;

size_t hess_part_bytes(int prec, int n, int tgt_begin, int n_tgt, int plan_tgt) {
  if (use_sym_hess(prec, n, tgt_begin, n_tgt, plan_tgt))
    return (size_t)(hess_sym_grouped(n) ? 1 + 2 * kHessSymGroup : hess_sym_tiles(n)) * (size_t)n *
           4 * sizeof(float4);
  return (size_t)kMaxChunks * 4 * vec_bytes(prec) * (size_t)std::max(n_tgt, 1);
}

int hess_partials(const Device& dev, int prec, const void* rec, const void* adj, int n,
                  int tgt_begin, int n_tgt, const KernelConsts& kc, void* part,
                  int part_cap_chunks, cudaStream_t st, int plan_tgt) {
  if (use_sym_hess(prec, n, tgt_begin, n_tgt, plan_tgt)) {
    // (the caller sized part with hess_part_bytes)
    const int T = hess_sym_tiles(n);
    const float kap = (float)kc.kappa;
    const float c1 = (float)(1.0 / (kc.kappa * kc.kappa * kc.s));
    const float a = (float)(kc.kappa * kc.c0[0]), b = (float)(kc.kappa * kc.c0[1]),
                c = (float)(kc.kappa * kc.c0[2]);
    if (!hess_sym_grouped(n)) {
      const dim3 grid((unsigned)T, (unsigned)(T / 2 + 1));
      if (hess_sym_tile(n) == kHessSymTileSmall)
        k_hess_sym_f32x2<4, 128, 3, 64><<<grid, 128, 0, st>>>(
            (const float4*)rec, (const float4*)adj, n, T, kap, a, b, c, c1, (float4*)part);
      else
        k_hess_sym_f32x2<6, 128, 2, 64><<<grid, 128, 0, st>>>(
            (const float4*)rec, (const float4*)adj, n, T, kap, a, b, c, c1, (float4*)part);
      return T;
    }
    float4* acc = (float4*)part;
    float4* slots = acc + 4 * (size_t)n;
    const int kend = T / 2 + 1;
    for (int k0 = 0; k0 < kend; k0 += kHessSymGroup) {
      const int k1 = std::min(kend, k0 + kHessSymGroup);
      if (hess_sym_tile(n) == kHessSymTileSmall)
        k_hess_sym_f32x2<4, 128, 3, 64><<<dim3((unsigned)T, (unsigned)(k1 - k0)), 128, 0, st>>>(
            (const float4*)rec, (const float4*)adj, n, T, kap, a, b, c, c1, slots, k0);
      else
        k_hess_sym_f32x2<6, 128, 2, 64><<<dim3((unsigned)T, (unsigned)(k1 - k0)), 128, 0, st>>>(
            (const float4*)rec, (const float4*)adj, n, T, kap, a, b, c, c1, slots, k0);
      k_fold_group4_f32<<<(n + 255) / 256, 256, 0, st>>>(slots, 2 * (k1 - k0), n, k0 == 0, acc);
    }
    return 1;
  }
  const int real_tgt = n_tgt;
  if (plan_tgt > 0) n_tgt = plan_tgt;
  if (prec == kF32) {
    static const int tpts[] = {4, 2, 1};
    static int occ = occupancy(k_hess_f32x2<4, kNT>, kNT);
    Plan pl = fit(plan(n, n_tgt, kNT, tpts, 3, kTile / 2, occ, dev.sms), real_tgt);
    if (pl.S > part_cap_chunks) return -1;
    n_tgt = real_tgt;
    static const bool packed = [] {
      const char* e = std::getenv("GS_HESS_PACKED");
      return e ? std::atoi(e) != 0 : true;
    }();
    if (packed && pl.tpt >= 2) {
      const float kap = (float)kc.kappa;
      const float c1 = (float)(1.0 / (kc.kappa * kc.kappa * kc.s));
      const float a = (float)(kc.kappa * kc.c0[0]), b = (float)(kc.kappa * kc.c0[1]),
                  c = (float)(kc.kappa * kc.c0[2]);
      if (pl.tpt == 4)
        k_hess_f32x2<4, kNT><<<pl.grid, kNT, 0, st>>>((const float4*)rec, (const float4*)adj, n, tgt_begin, n_tgt, pl.chunk, kap, a, b, c, c1, (float4*)part);
      else
        k_hess_f32x2<2, kNT><<<pl.grid, kNT, 0, st>>>((const float4*)rec, (const float4*)adj, n, tgt_begin, n_tgt, pl.chunk, kap, a, b, c, c1, (float4*)part);
      return pl.S;
    }
    const float kap = (float)kc.kappa;
    const float c1 = (float)(1.0 / (kc.kappa * kc.kappa * kc.s));
    const float a = (float)(kc.kappa * kc.c0[0]), b = (float)(kc.kappa * kc.c0[1]),
                c = (float)(kc.kappa * kc.c0[2]);
    switch (pl.tpt) {
      case 4: k_hess_f32<4, kNT><<<pl.grid, kNT, 0, st>>>((const float4*)rec, (const float4*)adj, n, tgt_begin, n_tgt, pl.chunk, kap, a, b, c, c1, (float4*)part); break;
      case 2: k_hess_f32<2, kNT><<<pl.grid, kNT, 0, st>>>((const float4*)rec, (const float4*)adj, n, tgt_begin, n_tgt, pl.chunk, kap, a, b, c, c1, (float4*)part); break;
      default: k_hess_f32<1, kNT><<<pl.grid, kNT, 0, st>>>((const float4*)rec, (const float4*)adj, n, tgt_begin, n_tgt, pl.chunk, kap, a, b, c, c1, (float4*)part); break;
    }
    return pl.S;
  }
  static const int tpts[] = {2, 1};
  static int occ = occupancy(k_hess_f64<2, kNT>, kNT);
  Plan pl = fit(plan(n, n_tgt, kNT, tpts, 2, kTile / 4, occ, dev.sms), real_tgt);
  if (pl.S > part_cap_chunks) return -1;
  n_tgt = real_tgt;
  switch (pl.tpt) {
    case 2: k_hess_f64<2, kNT><<<pl.grid, kNT, 0, st>>>((const double4*)rec, (const double4*)adj, n, tgt_begin, n_tgt, pl.chunk, kc.inv_two_s, kc.inv_s, (double4*)part); break;
    default: k_hess_f64<1, kNT><<<pl.grid, kNT, 0, st>>>((const double4*)rec, (const double4*)adj, n, tgt_begin, n_tgt, pl.chunk, kc.inv_two_s, kc.inv_s, (double4*)part); break;
  }
  return pl.S;
}

int vel_partials(const Device& dev, int prec, const void* rec, int n, const void* ev, int m,
                 const KernelConsts& kc, void* part, int part_cap_chunks, cudaStream_t st) {
  if (prec == kF32) {
    static const int tpts[] = {8, 4, 2, 1};
    static int occ = occupancy(k_vel_f32x2<8, kNT>, kNT);
    Plan pl = plan(n, m, kNT, tpts, 4, kTile, occ, dev.sms);
    if (pl.S > part_cap_chunks) return -1;
    const float kap = (float)kc.kappa, a = (float)(kc.kappa * kc.c0[0]),
                b = (float)(kc.kappa * kc.c0[1]), c = (float)(kc.kappa * kc.c0[2]);
    const float4* r = (const float4*)rec;
    const float4* e = (const float4*)ev;
    float4* o = (float4*)part;
    switch (pl.tpt) {  // packed pairs of evaluation points; TPT 1 stays scalar
      case 8: k_vel_f32x2<8, kNT><<<pl.grid, kNT, 0, st>>>(r, n, e, m, pl.chunk, kap, a, b, c, o); break;
      case 4: k_vel_f32x2<4, kNT><<<pl.grid, kNT, 0, st>>>(r, n, e, m, pl.chunk, kap, a, b, c, o); break;
      case 2: k_vel_f32x2<2, kNT><<<pl.grid, kNT, 0, st>>>(r, n, e, m, pl.chunk, kap, a, b, c, o); break;
      default: k_vel_f32<1, kNT><<<pl.grid, kNT, 0, st>>>(r, n, e, m, pl.chunk, kap, a, b, c, o); break;
    }
    return pl.S;
  }
  static const int tpts[] = {4, 2, 1};
  static int occ = occupancy(k_vel_f64<4, kNT>, kNT);
  Plan pl = plan(n, m, kNT, tpts, 3, kTile / 2, occ, dev.sms);
  if (pl.S > part_cap_chunks) return -1;
  switch (pl.tpt) {
    case 4: k_vel_f64<4, kNT><<<pl.grid, kNT, 0, st>>>((const double4*)rec, n, (const double4*)ev, m, pl.chunk, kc.inv_two_s, (double4*)part); break;
    case 2: k_vel_f64<2, kNT><<<pl.grid, kNT, 0, st>>>((const double4*)rec, n, (const double4*)ev, m, pl.chunk, kc.inv_two_s, (double4*)part); break;
    default: k_vel_f64<1, kNT><<<pl.grid, kNT, 0, st>>>((const double4*)rec, n, (const double4*)ev, m, pl.chunk, kc.inv_two_s, (double4*)part); break;
  }
  return pl.S;
}

}  // namespace gsb
