// bh.h -- device octree (tree.cu) and Barnes-Hut traversal (bh.cu) interfaces.
#pragma once

#include <memory>
#include <vector>

#include "engine.h"

namespace gsb {

// Device octree with the reference's node semantics (octree.cpp:25-117),
// built from midpoint-replay Morton keys. Nodes in depth-first pre-order
// (children 0..7): a node's subtree is [idx, skip) and its points are the
// contiguous leaf-order positions [begin, end].
struct DevTree {
  int prec = kF64;
  int64_t n = 0, m = -1;  // m: node count (-1 = only known on the device, first[n])
  int64_t cap = 0;        // node slots allocated
  // per point (index order)
  DBuf key_hi, key_lo;  // u64
  // per leaf-order position
  DBuf perm;            // i32 point index
  DBuf skey_hi, skey_lo;
  DBuf lcp;             // i32 common digits with the next position
  DBuf first;           // i32 [n+1] pre-order index of the first node starting here
  DBuf srec;            // [n][2] V4<R>: scaled q' (FP32) / q (FP64), p
  DBuf squ;             // [n] V4<R>: unscaled q (gate queries, aggregates)
  DBuf sadj;            // [n][2] V4<R>: alpha, beta in leaf order
  // per node
  DBuf meta;            // int4 {skip, begin, end, leaf | level << 8}
  DBuf start;           // i32 start position of each node (k_nodes)
  DBuf parent;          // i32
  DBuf nchild;          // i32
  DBuf outer;           // i32 outer (chunk-spanning) nodes + count (tree.cu aggregates)
  DBuf parts;           // per-chunk total / head / tail partial aggregates
  DBuf lo, hi;          // V4<R> tight AABB (unscaled)
  DBuf cen, mom;        // V4<R> centroid (scaled in FP32) + count / momentum sum + count bits
  DBuf nrec;            // [cap][4] V4<R> traversal record {centroid|point, code} {momentum|p, begin} {lo, count} {hi}
  DBuf nadj;            // [cap][2] V4<R> {alpha sum, beta mean} per node
  DBuf psum, msum;      // double4 exact-order-independent aggregates
  DBuf asum, bsum;      // double4
  DBuf root;            // double[6] padded root box
  // radix-sort scratch
  DBuf tmp_k, tmp_v, tmp_v2, hist;
  DBuf tie_scr;         // k_tie_sort's digit counts (long runs of equal key_hi)
  DBuf tie_buf;         // k_tie_sort's second code buffer
  DBuf klo_flag;        // u32: k_keys computed key_lo this build
  DBuf bbox_ctr;        // u32: k_bbox's arrival counter (self-resetting)
  DBuf scan_tmp;
  DBuf sm_ctr;          // i32 [1024] per-SM query-block counters of the walk (k_bh_ws)
  DBuf pq_win;          // u32 [windows][queries][3] per-window per-query counters (folded)
  DBuf scal;
  KernelConsts kc{};
  double thr = 0.0;
  bool adj_valid = false;
  // lean: the aggregates write only the traversal records (nrec / nadj), not
  // the FP64 node sums and boxes that downloads and rescales read -- set by
  // the flows, whose trees are only ever walked
  bool lean = false;
};

// root_box (host, {lo xyz, hi xyz}) overrides the padded bounding box
// (Octree(cell_min, cell_max) + insert, octree.hpp:38-51).
// overflow (device int, optional) is set when the tree needs more than the
// 4n + 64 node slots; the node count itself stays on the device.
int tree_build(const Device& dev, int prec, const KernelConsts& kc, const void* rec, int64_t n,
               DevTree& t, cudaStream_t st, const double* root_box = nullptr,
               int* overflow = nullptr);
// Morton (leaf) order of the points only: t.perm, t.srec (FP32 interaction
// coordinates, p) -- the locality order of the exact path's underflow cutoff.
int morton_order(const Device& dev, int prec, const KernelConsts& kc, const void* rec, int64_t n,
                 DevTree& t, cudaStream_t st);
// exact node count (host round trip on first call after a build)
int64_t tree_node_count(DevTree& t, cudaStream_t st);
// (re)writes the interaction coordinates (FP32: scaled by kc.kappa) and centroids
int tree_rescale(int prec, DevTree& t, const void* rec, const KernelConsts& kc, cudaStream_t st);
// adj: [n][2] records (alpha, beta) by point index; node sums + leaf-order copy
int tree_accumulate(int prec, DevTree& t, const void* adj, cudaStream_t st);
// leaf-order copy of per-point adjoints only (node sums untouched)
int tree_set_point_adjoints(int prec, DevTree& t, const void* adj, cudaStream_t st);
// host copies for gs_tree_download
int tree_download(DevTree& t, cudaStream_t st, int32_t* order, uint64_t* key_hi,
                  uint64_t* key_lo, int32_t* level, int32_t* parent, int32_t* skip,
                  int32_t* range, double* boxes, double* sums, uint32_t* count);

enum BhMode { kBhRhs = 0, kBhHess = 1, kBhVel = 2 };

struct BhQuery {
  int mode = kBhRhs;
  // RHS / HESS: queries are the tree's own points restricted to point indices
  // [tgt_begin, tgt_begin + n_tgt); partials written per target (index - tgt_begin)
  int tgt_begin = 0, n_tgt = 0;
  // VEL: m external eval records (x, -) ; partials per eval point.
  // by_index RHS / HESS: n_tgt external query records (x, px) at ev and, for
  // HESS, (alpha_i, beta_i) at eadj (a flow shard's own targets, or arbitrary
  // queries of bh_point_gradients / bh_point_hessian_products)
  const void* ev = nullptr;
  const void* eadj = nullptr;
  int m = 0;
  void* part = nullptr;
  uint32_t* per_query = nullptr;  // optional [nq][3] direct, approx, visited (query order)
  unsigned long long* totals = nullptr;  // optional [3] sums
  int ntask = 1;  // node windows (bh_tasks); part holds [ntask][queries] partials
  int lmd = 0;    // literal-mean-dot dot scale (RHS also sums c into the B partial's .w)
  int by_index = 0;  // RHS/HESS: queries = the n_tgt records at ev, not the tree's points
  int dense = 0;     // bh_tasks: 1 dense near fields (32 windows), 2 very dense (group walk)
};
int bh_tasks(int64_t nq, int64_t n, double thr, const KernelConsts& kc, int* dense = nullptr);
// host threads driving flows on one GPU at once (batched subjects); per thread
void set_bh_concurrency(int c);
// process-wide walk override (gs_set_bh_walk): kernel 0 by regime / 1 independent /
// 3 group / 4 split, tasks 0 auto / K windows; -1 restores the environment's choice
void set_bh_walk(int kernel, int tasks);
int bh_traverse(const Device& dev, int prec, DevTree& t, double sigma, double thr,
                const BhQuery& q, cudaStream_t st);

// Barnes-Hut work area of a flow: the current tree plus, for evaluate(), the
// forward trees kept per step (shooting.cpp:96-97, :177-183).
struct BhWork {
  DevTree cur;
  std::vector<std::unique_ptr<DevTree>> kept;
  int cache_slot = -1;
  DBuf part;   // traversal partials
  DBuf stats;  // u64 totals (direct, approximated, visited)
};

int bh_keep_trees(BhWork& w, int T);
int bh_forward_stage(const Device& dev, int prec, const KernelConsts& kc, const gs_config& cfg,
                     const void* rec, int64_t n, int64_t tb, int64_t nt, BhWork& w, FwdEpi e,
                     cudaStream_t st, int64_t* launches, int* energy_blocks, gs_stats* stats);
// adj: the full (alpha, beta) records (node sums); targets [tb, tb + nt)
int bh_backward_step(const Device& dev, int prec, const KernelConsts& kc, const gs_config& cfg,
                     const void* rec_k, void* adj, int64_t n, int64_t tb, int64_t nt, int k,
                     BhWork& w, bool cached, BwdEpi e, cudaStream_t st, gs_stats* stats);
int bh_velocity_step(const Device& dev, int prec, const KernelConsts& kc, const gs_config& cfg,
                     const void* rec_k, int64_t n, void* ev, int64_t m, BhWork& w, VelEpi e,
                     cudaStream_t st);

// Largest double T2 with sqrt(T2) <= thr: the gate sqrt(d2) > thr
// (octree.cpp:141-149 + bh_kernel.cpp:46) is then exactly d2 > T2.
double gate_t2(double thr);

}  // namespace gsb
