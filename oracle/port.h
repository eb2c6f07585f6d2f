/* TEST INFRASTRUCTURE ONLY -- the CPU oracle ("port"): a plain-C restatement
 * of the reference hot path (/root/reference/proj), used by tests/, smoke()
 * and bench.py's cpu_baseline leg as the CHECKER. Never linked into or called
 * by the product (paper_1907_04834_b200/).
 *
 * All arrays are AoS double[3*n] (the reference's std::vector<Vec3> layout,
 * core.hpp:16-20). Status codes follow include/geoshoot_b200.h.
 */
#ifndef GEOSHOOT_ORACLE_PORT_H
#define GEOSHOOT_ORACLE_PORT_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- kernel_exact.cpp ---------------------------------------------------- */
double port_hamiltonian(int64_t n, const double* q, const double* p, double sigma);
double port_exact_rhs(int64_t n, const double* q, const double* p, double sigma,
                      double* dHdp, double* dHdq);
void port_exact_velocity(int64_t m, const double* x, int64_t n, const double* q,
                         const double* p, double sigma, double* v);
void port_hessian_products(int64_t n, const double* q, const double* p,
                           const double* alpha, const double* beta, double sigma,
                           double* pq, double* pp, double* qq, double* qp);

/* ---- octree.cpp ---------------------------------------------------------- */
typedef struct port_tree port_tree;
port_tree* port_tree_build(int64_t n, const double* q, const double* p);
void port_tree_free(port_tree* t);
int64_t port_tree_node_count(const port_tree* t);
/* same flat layout as oracle/ref_capi.cpp:ref_tree_dump */
void port_tree_dump(const port_tree* t, double* boxes, double* sums, int32_t* ints,
                    int32_t* next_point);
void port_tree_accumulate(port_tree* t, const double* alpha, const double* beta);
/* Leaf order of a depth-first walk, children 0..7, bucket members ascending. */
void port_tree_leaf_order(const port_tree* t, int32_t* order);
/* Root box of Octree::build (bbox padded by 1e-9 * extent per axis). */
void port_root_box(int64_t n, const double* q, double* lo3, double* hi3);
/* Midpoint-replay digits (octree.cpp octant_of/make_child) from the root box:
 * key_hi holds levels 1..21 (63 bits, level 1 most significant), key_lo levels
 * 22..32 (33 bits). Digit = xbit | ybit<<1 | zbit<<2. */
void port_morton_keys(int64_t n, const double* q, const double* lo3, const double* hi3,
                      uint64_t* key_hi, uint64_t* key_lo);

/* ---- bh_kernel.cpp ------------------------------------------------------- */
/* per_query (optional): n x 3 u64 = direct, approximated, visited. */
void port_bh_rhs(const port_tree* t, int64_t n, const double* q, const double* p,
                 double sigma, double thr, int threads, double* dHdp, double* dHdq,
                 uint64_t* per_query);
void port_bh_hessprod(const port_tree* t, int64_t n, const double* q, const double* p,
                      const double* alpha, const double* beta, double sigma, double thr,
                      int threads, double* pq, double* pp, double* qq, double* qp);
void port_bh_velocity(const port_tree* t, int64_t m, const double* x, double sigma,
                      double thr, int threads, double* v, uint64_t* per_query);

/* ---- shooting.cpp (+ RK4 composed over the same RHS) --------------------- */
enum { PORT_EULER = 0, PORT_RK4 = 1 };
/* traj_q/traj_p: (T+1) x n x 3 (may be NULL when final_q/final_p given).
 * energy_out: 1/2 <p0, dH/dp(q0,p0)>. Returns 0 or 3 (non-finite; *bad_step set). */
int port_shoot_forward(int64_t n, const double* q0, const double* p0, double sigma,
                       int timesteps, int backend, double thr_mult, int integrator,
                       int threads, double* traj_q, double* traj_p, double* final_q,
                       double* final_p, double* energy_out, int* bad_step);
/* evaluate(): Euler forward keeping trees + adjoint backward. report[4] =
 * energy, attachment, total, sse. */
int port_evaluate(int64_t n, const double* q0, const double* p0, const double* target,
                  double sigma, double lambda, int timesteps, int backend, double thr_mult,
                  int threads, double* report, double* grad, int* bad_step);
int port_warp(int64_t n, int timesteps, const double* traj_q, const double* traj_p,
              int64_t m, const double* x, double sigma, int backend, double thr_mult,
              int threads, double* y, int* bad_step);

#ifdef __cplusplus
}
#endif
#endif
