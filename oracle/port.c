/* TEST INFRASTRUCTURE ONLY -- CPU oracle ("port") for the geodesic-shooting
 * hot path. It restates, in plain C, the reference algorithm of
 * /root/reference/proj (file:line cited per function) with the same operation
 * order, so that on identical FP64 inputs it reproduces the reference results
 * bit for bit (pinned against oracle/_ref in tests/test_oracle.py). It also
 * adds what the reference lacks but the parity contract needs:
 * the midpoint-replay Morton keys / DFS leaf order, and an RK4 integrator
 * composed over the reference RHS (tree rebuilt at every stage).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * this library; the product never does.
 */
#include "port.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double x, y, z; } v3;

static inline v3 ld(const double* a, int64_t i) { v3 r = {a[3 * i], a[3 * i + 1], a[3 * i + 2]}; return r; }
static inline void st(double* a, int64_t i, v3 v) { a[3 * i] = v.x; a[3 * i + 1] = v.y; a[3 * i + 2] = v.z; }
static inline v3 add(v3 a, v3 b) { v3 r = {a.x + b.x, a.y + b.y, a.z + b.z}; return r; }
static inline v3 sub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static inline v3 scl(double s, v3 a) { v3 r = {a.x * s, a.y * s, a.z * s}; return r; }
static inline double dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline double nrm2(v3 a) { return dot(a, a); }
static inline int finite3(v3 a) { return isfinite(a.x) && isfinite(a.y) && isfinite(a.z); }

/* ------------------------------------------------------------------------ */
/* tiny fork/join over query indices (parallel.hpp:16-34): contiguous chunks */
typedef struct {
  void (*fn)(void* ctx, int64_t i);
  void* ctx;
  int64_t lo, hi;
} chunk_t;

static void* run_chunk(void* a) {
  chunk_t* c = (chunk_t*)a;
  for (int64_t i = c->lo; i < c->hi; ++i) c->fn(c->ctx, i);
  return NULL;
}

static void par_for(int64_t n, int threads, void (*fn)(void*, int64_t), void* ctx) {
  if (threads <= 1 || n < 2) {
    for (int64_t i = 0; i < n; ++i) fn(ctx, i);
    return;
  }
  if (threads > n) threads = (int)n;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  chunk_t* ch = (chunk_t*)malloc(sizeof(chunk_t) * threads);
  for (int w = 0; w < threads; ++w) {
    ch[w].fn = fn; ch[w].ctx = ctx;
    ch[w].lo = n * w / threads; ch[w].hi = n * (w + 1) / threads;
    pthread_create(&th[w], NULL, run_chunk, &ch[w]);
  }
  for (int w = 0; w < threads; ++w) pthread_join(th[w], NULL);
  free(th); free(ch);
}

/* ------------------------------------------------------------------------ */
/* kernel_exact.cpp */

/* kernel_exact.cpp:13-27: diagonal first, then 2 * upper triangle */
double port_hamiltonian(int64_t n, const double* q, const double* p, double sigma) {
  const double inv_two_s = 1.0 / (2.0 * sigma * sigma);
  double h = 0.0;
  for (int64_t i = 0; i < n; ++i) h += dot(ld(p, i), ld(p, i));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) {
      const double g = exp(-nrm2(sub(ld(q, i), ld(q, j))) * inv_two_s);
      h += 2.0 * dot(ld(p, i), ld(p, j)) * g;
    }
  return h;
}

/* kernel_exact.cpp:29-61: symmetric i<j sweep scattering to both ends */
double port_exact_rhs(int64_t n, const double* q, const double* p, double sigma,
                      double* dHdp, double* dHdq) {
  const double s = sigma * sigma;
  const double inv_two_s = 1.0 / (2.0 * s);
  const double two_over_s = 2.0 / s;
  double h = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    st(dHdp, i, scl(2.0, ld(p, i)));
    v3 z = {0, 0, 0};
    st(dHdq, i, z);
    h += dot(ld(p, i), ld(p, i));
  }
  for (int64_t i = 0; i < n; ++i) {
    const v3 qi = ld(q, i), pi = ld(p, i);
    v3 api = ld(dHdp, i), aqi = ld(dHdq, i);
    for (int64_t j = i + 1; j < n; ++j) {
      const v3 pj = ld(p, j);
      const v3 d = sub(qi, ld(q, j));
      const double g = exp(-nrm2(d) * inv_two_s);
      const double pipj = dot(pi, pj);
      api = add(api, scl(2.0 * g, pj));
      st(dHdp, j, add(ld(dHdp, j), scl(2.0 * g, pi)));
      const v3 grad = scl(two_over_s * pipj * g, d);
      aqi = sub(aqi, grad);
      st(dHdq, j, add(ld(dHdq, j), grad));
      h += 2.0 * pipj * g;
    }
    st(dHdp, i, api);
    st(dHdq, i, aqi);
  }
  return h;
}

/* kernel_exact.cpp:70-82 */
void port_exact_velocity(int64_t m, const double* x, int64_t n, const double* q,
                         const double* p, double sigma, double* v) {
  const double inv_two_s = 1.0 / (2.0 * sigma * sigma);
  for (int64_t e = 0; e < m; ++e) {
    v3 sum = {0, 0, 0};
    const v3 xe = ld(x, e);
    for (int64_t i = 0; i < n; ++i)
      sum = add(sum, scl(exp(-nrm2(sub(xe, ld(q, i))) * inv_two_s), ld(p, i)));
    st(v, e, sum);
  }
}

/* kernel_exact.cpp:84-135 */
void port_hessian_products(int64_t n, const double* q, const double* p,
                           const double* alpha, const double* beta, double sigma,
                           double* pq, double* pp, double* qq, double* qp) {
  const double s = sigma * sigma;
  const double inv_s = 1.0 / s;
  const double inv_two_s = 0.5 * inv_s;
  const double two_over_s = 2.0 * inv_s;
  const v3 z = {0, 0, 0};
  for (int64_t i = 0; i < n; ++i) {
    st(pq, i, z); st(qq, i, z); st(qp, i, z);
    st(pp, i, scl(2.0, ld(alpha, i)));
  }
  for (int64_t i = 0; i < n; ++i) {
    const v3 qi = ld(q, i), pi = ld(p, i), ai = ld(alpha, i), bi = ld(beta, i);
    for (int64_t j = i + 1; j < n; ++j) {
      const v3 pj = ld(p, j), aj = ld(alpha, j);
      const v3 d = sub(qi, ld(q, j));
      const double g = exp(-nrm2(d) * inv_two_s);
      const v3 db = sub(bi, ld(beta, j));
      const double d_db = dot(d, db);

      const double uc = two_over_s * g * (dot(pj, ai) + dot(pi, aj));
      st(pq, i, sub(ld(pq, i), scl(uc, d)));
      st(pq, j, add(ld(pq, j), scl(uc, d)));

      st(pp, i, add(ld(pp, i), scl(2.0 * g, aj)));
      st(pp, j, add(ld(pp, j), scl(2.0 * g, ai)));

      const double zc = two_over_s * g * dot(pi, pj);
      const v3 zterm = sub(scl(d_db * inv_s, d), db);
      st(qq, i, add(ld(qq, i), scl(zc, zterm)));
      st(qq, j, sub(ld(qq, j), scl(zc, zterm)));

      const double mc = two_over_s * g * d_db;
      st(qp, i, sub(ld(qp, i), scl(mc, pj)));
      st(qp, j, sub(ld(qp, j), scl(mc, pi)));
    }
  }
}

/* ------------------------------------------------------------------------ */
/* octree.cpp -- pointer-free restatement with the same node semantics       */

enum { MAX_DEPTH = 32, NO_CHILD = -1 };

typedef struct {
  v3 cmin, cmax, amin, amax, psum, msum, asum, bsum;
  uint32_t count;
  int32_t child[8];
  int32_t first;
  int leaf;
} pnode;

struct port_tree {
  pnode* nodes;
  int64_t n_nodes, cap;
  int64_t n_points;
  double* q;  /* copies, index order (octree.hpp:83-86) */
  double* p;
  int32_t* next;
};

static int32_t new_node(port_tree* t, v3 lo, v3 hi) {
  if (t->n_nodes == t->cap) {
    t->cap = t->cap ? 2 * t->cap : 64;
    t->nodes = (pnode*)realloc(t->nodes, sizeof(pnode) * t->cap);
  }
  pnode* nd = &t->nodes[t->n_nodes];
  memset(nd, 0, sizeof *nd);
  nd->cmin = lo; nd->cmax = hi;
  for (int c = 0; c < 8; ++c) nd->child[c] = NO_CHILD;
  nd->first = -1;
  nd->leaf = 1;
  return (int32_t)t->n_nodes++;
}

/* octree.cpp:42-45 -- ties go high */
static int octant(const pnode* nd, v3 x) {
  const v3 c = scl(0.5, add(nd->cmin, nd->cmax));
  return (x.x >= c.x ? 1 : 0) | (x.y >= c.y ? 2 : 0) | (x.z >= c.z ? 4 : 0);
}

/* octree.cpp:47-57 */
static void stats_add(pnode* nd, v3 q, v3 p) {
  if (nd->count == 0) {
    nd->amin = nd->amax = q;
  } else {
    nd->amin.x = nd->amin.x < q.x ? nd->amin.x : q.x;
    nd->amin.y = nd->amin.y < q.y ? nd->amin.y : q.y;
    nd->amin.z = nd->amin.z < q.z ? nd->amin.z : q.z;
    nd->amax.x = nd->amax.x > q.x ? nd->amax.x : q.x;
    nd->amax.y = nd->amax.y > q.y ? nd->amax.y : q.y;
    nd->amax.z = nd->amax.z > q.z ? nd->amax.z : q.z;
  }
  nd->psum = add(nd->psum, q);
  nd->msum = add(nd->msum, p);
  nd->count++;
}

/* octree.cpp:59-72 -- child cell from the parent midpoint */
static int32_t child_of(port_tree* t, int32_t parent, int oct) {
  const v3 lo = t->nodes[parent].cmin, hi = t->nodes[parent].cmax;
  const v3 c = scl(0.5, add(lo, hi));
  v3 a = {oct & 1 ? c.x : lo.x, oct & 2 ? c.y : lo.y, oct & 4 ? c.z : lo.z};
  v3 b = {oct & 1 ? hi.x : c.x, oct & 2 ? hi.y : c.y, oct & 4 ? hi.z : c.z};
  const int32_t idx = new_node(t, a, b);
  t->nodes[parent].child[oct] = idx;
  return idx;
}

/* octree.cpp:74-117 -- sequential insertion, single-point leaves, bucket at
 * depth 32, statistics updated on the way down */
static void insert_point(port_tree* t, int32_t index, v3 x, v3 m) {
  int32_t cur = 0;
  int depth = 0;
  stats_add(&t->nodes[0], x, m);
  for (;;) {
    pnode* nd = &t->nodes[cur];
    if (nd->leaf) {
      if (nd->count == 1) { nd->first = index; return; }
      if (depth == MAX_DEPTH) {
        t->next[index] = nd->first;
        nd->first = index;
        return;
      }
      const int32_t occ = nd->first;
      nd->first = -1;
      nd->leaf = 0;
      const v3 oq = ld(t->q, occ), op = ld(t->p, occ);
      const int32_t ch = child_of(t, cur, octant(&t->nodes[cur], oq));
      stats_add(&t->nodes[ch], oq, op);
      t->nodes[ch].first = occ;
    }
    const int oc = octant(&t->nodes[cur], x);
    int32_t ch = t->nodes[cur].child[oc];
    if (ch == NO_CHILD) ch = child_of(t, cur, oc);
    cur = ch;
    ++depth;
    stats_add(&t->nodes[cur], x, m);
  }
}

/* octree.cpp:9,25-40 */
void port_root_box(int64_t n, const double* q, double* lo3, double* hi3) {
  v3 lo = ld(q, 0), hi = ld(q, 0);
  for (int64_t i = 0; i < n; ++i) {
    const v3 x = ld(q, i);
    lo.x = lo.x < x.x ? lo.x : x.x; lo.y = lo.y < x.y ? lo.y : x.y; lo.z = lo.z < x.z ? lo.z : x.z;
    hi.x = hi.x > x.x ? hi.x : x.x; hi.y = hi.y > x.y ? hi.y : x.y; hi.z = hi.z > x.z ? hi.z : x.z;
  }
  const v3 pad = scl(1e-9, sub(hi, lo));
  st(lo3, 0, sub(lo, pad));
  st(hi3, 0, add(hi, pad));
}

port_tree* port_tree_build(int64_t n, const double* q, const double* p) {
  port_tree* t = (port_tree*)calloc(1, sizeof *t);
  double lo[3], hi[3];
  port_root_box(n, q, lo, hi);
  new_node(t, ld(lo, 0), ld(hi, 0));
  t->n_points = n;
  t->q = (double*)malloc(sizeof(double) * 3 * n);
  t->p = (double*)malloc(sizeof(double) * 3 * n);
  t->next = (int32_t*)malloc(sizeof(int32_t) * n);
  memcpy(t->q, q, sizeof(double) * 3 * n);
  memcpy(t->p, p, sizeof(double) * 3 * n);
  for (int64_t i = 0; i < n; ++i) {
    t->next[i] = -1;
    insert_point(t, (int32_t)i, ld(q, i), ld(p, i));
  }
  return t;
}

void port_tree_free(port_tree* t) {
  if (!t) return;
  free(t->nodes); free(t->q); free(t->p); free(t->next); free(t);
}

int64_t port_tree_node_count(const port_tree* t) { return t->n_nodes; }

void port_tree_dump(const port_tree* t, double* boxes, double* sums, int32_t* ints,
                    int32_t* next_point) {
  for (int64_t k = 0; k < t->n_nodes; ++k) {
    const pnode* nd = &t->nodes[k];
    const v3 b[4] = {nd->cmin, nd->cmax, nd->amin, nd->amax};
    const v3 s[4] = {nd->psum, nd->msum, nd->asum, nd->bsum};
    memcpy(boxes + 12 * k, b, sizeof b);
    memcpy(sums + 12 * k, s, sizeof s);
    int32_t* o = ints + 11 * k;
    o[0] = (int32_t)nd->count;
    for (int c = 0; c < 8; ++c) o[1 + c] = nd->child[c];
    o[9] = nd->first;
    o[10] = nd->leaf;
  }
  for (int64_t i = 0; i < t->n_points; ++i) next_point[i] = t->next[i];
}

/* octree.cpp:119-139 -- zero, then re-sum along each point's root->leaf path */
void port_tree_accumulate(port_tree* t, const double* alpha, const double* beta) {
  const v3 z = {0, 0, 0};
  for (int64_t k = 0; k < t->n_nodes; ++k) t->nodes[k].asum = t->nodes[k].bsum = z;
  for (int64_t i = 0; i < t->n_points; ++i) {
    int32_t cur = 0;
    for (;;) {
      pnode* nd = &t->nodes[cur];
      nd->asum = add(nd->asum, ld(alpha, i));
      nd->bsum = add(nd->bsum, ld(beta, i));
      if (nd->leaf) break;
      cur = nd->child[octant(nd, ld(t->q, i))];
    }
  }
}

static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

static void leaf_order_rec(const port_tree* t, int32_t k, int32_t* order, int64_t* pos) {
  const pnode* nd = &t->nodes[k];
  if (nd->leaf) {
    const int64_t start = *pos;
    for (int32_t i = nd->first; i >= 0; i = t->next[i]) order[(*pos)++] = i;
    qsort(order + start, (size_t)(*pos - start), sizeof(int32_t), cmp_i32);
    return;
  }
  for (int c = 0; c < 8; ++c)
    if (nd->child[c] != NO_CHILD) leaf_order_rec(t, nd->child[c], order, pos);
}

void port_tree_leaf_order(const port_tree* t, int32_t* order) {
  int64_t pos = 0;
  leaf_order_rec(t, 0, order, &pos);
}

/* Morton digits by replaying octant_of/make_child per axis.
 * The per-axis recursions are independent, so each axis is replayed alone. */
void port_morton_keys(int64_t n, const double* q, const double* lo3, const double* hi3,
                      uint64_t* key_hi, uint64_t* key_lo) {
  for (int64_t i = 0; i < n; ++i) {
    uint64_t kh = 0, kl = 0;
    double lo[3] = {lo3[0], lo3[1], lo3[2]}, hi[3] = {hi3[0], hi3[1], hi3[2]};
    for (int lev = 1; lev <= MAX_DEPTH; ++lev) {
      unsigned dig = 0;
      for (int a = 0; a < 3; ++a) {
        const double c = 0.5 * (lo[a] + hi[a]);
        const int bit = q[3 * i + a] >= c;
        if (bit) lo[a] = c; else hi[a] = c;
        dig |= (unsigned)bit << a;
      }
      if (lev <= 21) kh = (kh << 3) | dig;
      else kl = (kl << 3) | dig;
    }
    key_hi[i] = kh;
    key_lo[i] = kl;
  }
}

/* ------------------------------------------------------------------------ */
/* bh_kernel.cpp -- LIFO stack traversal, leaf first, gate, push 0..7        */

/* octree.cpp:141-149 */
static double min_dist(const pnode* nd, v3 x) {
  double dx = nd->amin.x - x.x, dy = nd->amin.y - x.y, dz = nd->amin.z - x.z;
  const double ex = x.x - nd->amax.x, ey = x.y - nd->amax.y, ez = x.z - nd->amax.z;
  /* std::max({a, 0.0, b}) */
  dx = dx < 0.0 ? 0.0 : dx; dx = dx < ex ? ex : dx;
  dy = dy < 0.0 ? 0.0 : dy; dy = dy < ey ? ey : dy;
  dz = dz < 0.0 ? 0.0 : dz; dz = dz < ez ? ez : dz;
  return sqrt(dx * dx + dy * dy + dz * dz);
}

static v3 centroid(const pnode* nd) { return scl(1.0 / nd->count, nd->psum); }

enum { STACK_CAP = 8 * (MAX_DEPTH + 1) };

typedef struct {
  const port_tree* t;
  const double *q, *p, *alpha, *beta;
  double sigma, thr;
  double *o1, *o2, *o3, *o4;
  uint64_t* per_query;
} bh_job;

/* bh_kernel.cpp:81-112 over one query */
static void bh_grad_one(void* ctx, int64_t i) {
  const bh_job* J = (const bh_job*)ctx;
  const port_tree* t = J->t;
  const double s = J->sigma * J->sigma;
  const double inv_two_s = 0.5 / s;
  const double two_over_s = 2.0 / s;
  const v3 x = ld(J->q, i), px = ld(J->p, i);
  v3 dp = {0, 0, 0}, dq = {0, 0, 0};
  uint64_t nd_direct = 0, nd_approx = 0, nd_visit = 0;
  int32_t stack[STACK_CAP];
  int top = 0;
  stack[top++] = 0;
  while (top > 0) {
    const pnode* nd = &t->nodes[stack[--top]];
    ++nd_visit;
    if (nd->leaf) {
      for (int32_t j = nd->first; j >= 0; j = t->next[j]) {
        const v3 pj = ld(t->p, j);
        const v3 d = sub(x, ld(t->q, j));
        const double g = exp(-nrm2(d) * inv_two_s);
        dp = add(dp, scl(2.0 * g, pj));
        dq = sub(dq, scl(two_over_s * dot(px, pj) * g, d));
        ++nd_direct;
      }
    } else if (min_dist(nd, x) > J->thr) {
      const v3 d = sub(x, centroid(nd));
      const double g = exp(-nrm2(d) * inv_two_s);
      dp = add(dp, scl(2.0 * g, nd->msum));
      dq = sub(dq, scl(two_over_s * (dot(px, nd->msum) * 1.0) * g, d));
      ++nd_approx;
    } else {
      for (int c = 0; c < 8; ++c)
        if (nd->child[c] != NO_CHILD) stack[top++] = nd->child[c];
    }
  }
  st(J->o1, i, dp);
  st(J->o2, i, dq);
  if (J->per_query) {
    J->per_query[3 * i] = nd_direct;
    J->per_query[3 * i + 1] = nd_approx;
    J->per_query[3 * i + 2] = nd_visit;
  }
}

void port_bh_rhs(const port_tree* t, int64_t n, const double* q, const double* p,
                 double sigma, double thr, int threads, double* dHdp, double* dHdq,
                 uint64_t* per_query) {
  bh_job J = {t, q, p, NULL, NULL, sigma, thr, dHdp, dHdq, NULL, NULL, per_query};
  par_for(n, threads, bh_grad_one, &J);
}

/* bh_kernel.cpp:114-160 over one query */
static void bh_hess_one(void* ctx, int64_t i) {
  const bh_job* J = (const bh_job*)ctx;
  const port_tree* t = J->t;
  const double s = J->sigma * J->sigma;
  const double inv_s = 1.0 / s;
  const double inv_two_s = 0.5 * inv_s;
  const double two_over_s = 2.0 * inv_s;
  const v3 qi = ld(J->q, i), pi = ld(J->p, i), ai = ld(J->alpha, i), bi = ld(J->beta, i);
  v3 pq = {0, 0, 0}, pp = {0, 0, 0}, qq = {0, 0, 0}, qp = {0, 0, 0};
  int32_t stack[STACK_CAP];
  int top = 0;
  stack[top++] = 0;
  while (top > 0) {
    const pnode* nd = &t->nodes[stack[--top]];
    if (nd->leaf) {
      for (int32_t j = nd->first; j >= 0; j = t->next[j]) {
        const v3 pj = ld(t->p, j), aj = ld(J->alpha, j);
        const v3 d = sub(qi, ld(t->q, j));
        const double g = exp(-nrm2(d) * inv_two_s);
        const v3 db = sub(bi, ld(J->beta, j));
        const double d_db = dot(d, db);
        pq = sub(pq, scl(two_over_s * g * (dot(pj, ai) + dot(pi, aj)), d));
        pp = add(pp, scl(2.0 * g, aj));
        qq = add(qq, scl(two_over_s * g * dot(pi, pj), sub(scl(d_db * inv_s, d), db)));
        qp = sub(qp, scl(two_over_s * g * d_db, pj));
      }
    } else if (min_dist(nd, qi) > J->thr) {
      const v3 d = sub(qi, centroid(nd));
      const double g = exp(-nrm2(d) * inv_two_s);
      const v3 db = sub(bi, scl(1.0 / nd->count, nd->bsum));
      const double d_db = dot(d, db);
      pq = sub(pq, scl(two_over_s * g * (dot(nd->msum, ai) + dot(pi, nd->asum)), d));
      pp = add(pp, scl(2.0 * g, nd->asum));
      qq = add(qq, scl(two_over_s * g * (dot(pi, nd->msum) * 1.0), sub(scl(d_db * inv_s, d), db)));
      qp = sub(qp, scl(two_over_s * g * d_db, nd->msum));
    } else {
      for (int c = 0; c < 8; ++c)
        if (nd->child[c] != NO_CHILD) stack[top++] = nd->child[c];
    }
  }
  st(J->o1, i, pq); st(J->o2, i, pp); st(J->o3, i, qq); st(J->o4, i, qp);
}

void port_bh_hessprod(const port_tree* t, int64_t n, const double* q, const double* p,
                      const double* alpha, const double* beta, double sigma, double thr,
                      int threads, double* pq, double* pp, double* qq, double* qp) {
  bh_job J = {t, q, p, alpha, beta, sigma, thr, pq, pp, qq, qp, NULL};
  par_for(n, threads, bh_hess_one, &J);
}

/* bh_kernel.cpp:62-79 over one eval point */
static void bh_vel_one(void* ctx, int64_t e) {
  const bh_job* J = (const bh_job*)ctx;
  const port_tree* t = J->t;
  const double inv_two_s = 1.0 / (2.0 * J->sigma * J->sigma);
  const v3 x = ld(J->q, e);
  v3 v = {0, 0, 0};
  uint64_t c_d = 0, c_a = 0, c_v = 0;
  int32_t stack[STACK_CAP];
  int top = 0;
  stack[top++] = 0;
  while (top > 0) {
    const pnode* nd = &t->nodes[stack[--top]];
    ++c_v;
    if (nd->leaf) {
      for (int32_t j = nd->first; j >= 0; j = t->next[j]) {
        v = add(v, scl(exp(-nrm2(sub(x, ld(t->q, j))) * inv_two_s), ld(t->p, j)));
        ++c_d;
      }
    } else if (min_dist(nd, x) > J->thr) {
      v = add(v, scl(exp(-nrm2(sub(x, centroid(nd))) * inv_two_s), nd->msum));
      ++c_a;
    } else {
      for (int c = 0; c < 8; ++c)
        if (nd->child[c] != NO_CHILD) stack[top++] = nd->child[c];
    }
  }
  st(J->o1, e, v);
  if (J->per_query) {
    J->per_query[3 * e] = c_d; J->per_query[3 * e + 1] = c_a; J->per_query[3 * e + 2] = c_v;
  }
}

void port_bh_velocity(const port_tree* t, int64_t m, const double* x, double sigma,
                      double thr, int threads, double* v, uint64_t* per_query) {
  bh_job J = {t, x, NULL, NULL, NULL, sigma, thr, v, NULL, NULL, NULL, per_query};
  par_for(m, threads, bh_vel_one, &J);
}

/* ------------------------------------------------------------------------ */
/* shooting.cpp                                                              */

/* step_gradients, shooting.cpp:31-60 (tree built from the same state) */
static void rhs(int64_t n, const double* q, const double* p, double sigma, int backend,
                double thr, int threads, double* dHdp, double* dHdq) {
  if (!backend) {
    port_exact_rhs(n, q, p, sigma, dHdp, dHdq);
    return;
  }
  port_tree* t = port_tree_build(n, q, p);
  port_bh_rhs(t, n, q, p, sigma, thr, threads, dHdp, dHdq, NULL);
  port_tree_free(t);
}

static int all_finite(int64_t n, const double* a) {
  for (int64_t i = 0; i < 3 * n; ++i) if (!isfinite(a[i])) return 0;
  return 1;
}

/* run_forward, shooting.cpp:68-124 (Euler) ; RK4 = classical four-stage
 * scheme with the stage combination written as in test_shooting.cpp:42-59 */
int port_shoot_forward(int64_t n, const double* q0, const double* p0, double sigma,
                       int timesteps, int backend, double thr_mult, int integrator,
                       int threads, double* traj_q, double* traj_p, double* final_q,
                       double* final_p, double* energy_out, int* bad_step) {
  const size_t b = sizeof(double) * 3 * n;
  const double dt = 1.0 / timesteps;
  const double thr = thr_mult * sigma;
  double* q = (double*)malloc(b); double* p = (double*)malloc(b);
  double* gp = (double*)malloc(b); double* gq = (double*)malloc(b);
  memcpy(q, q0, b); memcpy(p, p0, b);
  if (traj_q) { memcpy(traj_q, q0, b); memcpy(traj_p, p0, b); }
  double *kq[4], *kp[4], *yq = NULL, *yp = NULL;
  if (integrator == PORT_RK4) {
    for (int s = 0; s < 4; ++s) { kq[s] = (double*)malloc(b); kp[s] = (double*)malloc(b); }
    yq = (double*)malloc(b); yp = (double*)malloc(b);
  }
  int status = 0;
  for (int k = 0; k < timesteps; ++k) {
    if (integrator == PORT_EULER) {
      rhs(n, q, p, sigma, backend, thr, threads, gp, gq);
      if (k == 0 && energy_out) {
        double h = 0.0;
        for (int64_t i = 0; i < n; ++i) h += dot(ld(p0, i), ld(gp, i));
        *energy_out = 0.5 * h;
      }
      for (int64_t i = 0; i < n; ++i) {
        st(q, i, add(ld(q, i), scl(dt, ld(gp, i))));
        st(p, i, sub(ld(p, i), scl(dt, ld(gq, i))));
      }
    } else {
      static const double w[3] = {0.5, 0.5, 1.0};
      for (int s = 0; s < 4; ++s) {
        const double* sq = s == 0 ? q : yq;
        const double* sp = s == 0 ? p : yp;
        rhs(n, sq, sp, sigma, backend, thr, threads, kq[s], gq);
        if (k == 0 && s == 0 && energy_out) {
          double h = 0.0;
          for (int64_t i = 0; i < n; ++i) h += dot(ld(p0, i), ld(kq[0], i));
          *energy_out = 0.5 * h;
        }
        for (int64_t i = 0; i < 3 * n; ++i) kp[s][i] = -gq[i];
        if (s < 3) {
          const double hw = w[s] * dt;
          for (int64_t i = 0; i < 3 * n; ++i) {
            yq[i] = q[i] + hw * kq[s][i];
            yp[i] = p[i] + hw * kp[s][i];
          }
        }
      }
      const double h6 = dt / 6;
      for (int64_t i = 0; i < 3 * n; ++i) {
        q[i] += h6 * (kq[0][i] + 2 * kq[1][i] + 2 * kq[2][i] + kq[3][i]);
        p[i] += h6 * (kp[0][i] + 2 * kp[1][i] + 2 * kp[2][i] + kp[3][i]);
      }
    }
    if (!all_finite(n, q) || !all_finite(n, p)) {
      status = 3;
      if (bad_step) *bad_step = k + 1;
      break;
    }
    if (traj_q) {
      memcpy(traj_q + (size_t)(k + 1) * 3 * n, q, b);
      memcpy(traj_p + (size_t)(k + 1) * 3 * n, p, b);
    }
  }
  if (final_q) memcpy(final_q, q, b);
  if (final_p) memcpy(final_p, p, b);
  if (integrator == PORT_RK4) {
    for (int s = 0; s < 4; ++s) { free(kq[s]); free(kp[s]); }
    free(yq); free(yp);
  }
  free(q); free(p); free(gp); free(gq);
  return status;
}

/* evaluate, shooting.cpp:302-314 = run_forward(keep_trees) + make_report
 * (:126-138) + run_backward (:143-240) reusing the forward trees */
int port_evaluate(int64_t n, const double* q0, const double* p0, const double* target,
                  double sigma, double lambda, int timesteps, int backend, double thr_mult,
                  int threads, double* report, double* grad, int* bad_step) {
  const size_t b = sizeof(double) * 3 * n;
  const double dt = 1.0 / timesteps;
  const double thr = thr_mult * sigma;
  double* tq = (double*)malloc(b * (timesteps + 1));
  double* tp = (double*)malloc(b * (timesteps + 1));
  port_tree** trees = (port_tree**)calloc((size_t)timesteps, sizeof(port_tree*));
  double* gp = (double*)malloc(b); double* gq = (double*)malloc(b);
  memcpy(tq, q0, b); memcpy(tp, p0, b);
  double energy = 0.0;
  int status = 0;
  for (int k = 0; k < timesteps && !status; ++k) {
    const double* q = tq + (size_t)k * 3 * n;
    const double* p = tp + (size_t)k * 3 * n;
    if (backend) {
      trees[k] = port_tree_build(n, q, p);
      port_bh_rhs(trees[k], n, q, p, sigma, thr, threads, gp, gq, NULL);
    } else {
      port_exact_rhs(n, q, p, sigma, gp, gq);
    }
    if (k == 0) {
      double h = 0.0;
      for (int64_t i = 0; i < n; ++i) h += dot(ld(p0, i), ld(gp, i));
      energy = 0.5 * h;
    }
    double* qn = tq + (size_t)(k + 1) * 3 * n;
    double* pn = tp + (size_t)(k + 1) * 3 * n;
    for (int64_t i = 0; i < n; ++i) {
      st(qn, i, add(ld(q, i), scl(dt, ld(gp, i))));
      st(pn, i, sub(ld(p, i), scl(dt, ld(gq, i))));
    }
    if (!all_finite(n, qn) || !all_finite(n, pn)) {
      status = 3;
      if (bad_step) *bad_step = k + 1;
    }
  }
  if (!status) {
    const double* q1 = tq + (size_t)timesteps * 3 * n;
    double sse = 0.0;
    for (int64_t i = 0; i < n; ++i) sse += nrm2(sub(ld(q1, i), ld(target, i)));
    report[0] = energy;
    report[3] = sse;
    report[1] = lambda * sse;
    report[2] = report[0] + report[1];

    double* al = (double*)malloc(b); double* be = (double*)calloc(3 * (size_t)n, sizeof(double));
    double *pq = (double*)malloc(b), *pp = (double*)malloc(b), *qq = (double*)malloc(b),
           *qp = (double*)malloc(b);
    for (int64_t i = 0; i < n; ++i) st(al, i, scl(2.0 * lambda, sub(ld(q1, i), ld(target, i))));
    for (int k = timesteps - 1; k >= 0; --k) {
      const double* q = tq + (size_t)k * 3 * n;
      const double* p = tp + (size_t)k * 3 * n;
      if (backend) {
        port_tree_accumulate(trees[k], al, be);
        port_bh_hessprod(trees[k], n, q, p, al, be, sigma, thr, threads, pq, pp, qq, qp);
      } else {
        port_hessian_products(n, q, p, al, be, sigma, pq, pp, qq, qp);
      }
      for (int64_t i = 0; i < n; ++i) {
        st(al, i, add(ld(al, i), scl(dt, sub(ld(pq, i), ld(qq, i)))));
        st(be, i, add(ld(be, i), scl(dt, sub(ld(pp, i), ld(qp, i)))));
      }
    }
    if (backend) port_bh_rhs(trees[0], n, q0, p0, sigma, thr, 1, gp, gq, NULL);
    else port_exact_rhs(n, q0, p0, sigma, gp, gq);
    for (int64_t i = 0; i < n; ++i) st(grad, i, add(ld(be, i), ld(gp, i)));
    free(al); free(be); free(pq); free(pp); free(qq); free(qp);
  }
  for (int k = 0; k < timesteps; ++k) port_tree_free(trees[k]);
  free(trees); free(tq); free(tp); free(gp); free(gq);
  return status;
}

/* warp_points, shooting.cpp:266-300 */
int port_warp(int64_t n, int timesteps, const double* traj_q, const double* traj_p,
              int64_t m, const double* x, double sigma, int backend, double thr_mult,
              int threads, double* y, int* bad_step) {
  const double dt = 1.0 / timesteps;
  const double thr = thr_mult * sigma;
  double* v = (double*)malloc(sizeof(double) * 3 * m);
  memcpy(y, x, sizeof(double) * 3 * m);
  for (int k = 0; k < timesteps; ++k) {
    const double* q = traj_q + (size_t)k * 3 * n;
    const double* p = traj_p + (size_t)k * 3 * n;
    if (backend) {
      port_tree* t = port_tree_build(n, q, p);
      port_bh_velocity(t, m, y, sigma, thr, threads, v, NULL);
      port_tree_free(t);
    } else {
      port_exact_velocity(m, y, n, q, p, sigma, v);
    }
    for (int64_t e = 0; e < m; ++e) st(y, e, add(ld(y, e), scl(dt, scl(2.0, ld(v, e)))));
    if (!all_finite(m, y)) {
      if (bad_step) *bad_step = k + 1;
      free(v);
      return 3;
    }
  }
  free(v);
  return 0;
}
