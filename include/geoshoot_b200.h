/*
 * geoshoot_b200.h -- C ABI of the B200-native geodesic-shooting hot path.
 *
 * This is the drop-in boundary. Every entry point takes plain
 * host pointers in the reference layout -- `const double* xyz` of 3*n doubles,
 * i.e. reinterpret_cast<const double*>(std::vector<Vec3>::data()), Vec3 being
 * three doubles (reference core.hpp:16-20) -- plus sizes, and returns a
 * gs_status. No C++ types, no torch types, no exceptions cross it. The C++
 * reference API (paper_1907_04834_b200/include/geoshoot/*.hpp) is a thin shim
 * over these calls that maps gs_status back to the reference's exception
 * types; INTEGRATION.md shows the binding a reference maintainer would add.
 *
 * Each function names the reference interface it replaces
 * (file:line under the reference's proj/).
 *
 * Calls are synchronous at the boundary: results are in host memory when the
 * call returns. One gs_ctx per host thread (a context owns a CUDA stream and
 * its workspaces). The device work is done by hand-written sm_100a kernels;
 * there is no CPU fallback: without a usable B200 gs_create fails with
 * GS_NO_DEVICE.
 */
#ifndef GEOSHOOT_B200_H
#define GEOSHOOT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_ABI_VERSION 1

/* Mirrors the reference's exception types (core.hpp:69-116). */
typedef enum gs_status {
  GS_OK = 0,
  GS_DIMENSION_MISMATCH = 1, /* DimensionMismatch, core.hpp:69 / require_aligned :172-178 */
  GS_CONFIG_ERROR = 2,       /* ConfigError{violations}, core.hpp:233-247 (mask: gs_last_config_violations) */
  GS_NONFINITE = 3,          /* NonFiniteState{timestep}, core.hpp:83-89 (step: gs_last_nonfinite_step) */
  GS_CONFIG_MISMATCH = 4,    /* ConfigMismatch, core.hpp:91 */
  GS_EMPTY_TREE = 5,         /* EmptyTree, core.hpp:77 */
  GS_OUT_OF_BOUNDS = 6,      /* OutOfBounds, core.hpp:73 */
  GS_INVALID_ARGUMENT = 7,   /* std::invalid_argument (empty / non-finite PointSet, core.hpp:124-170) */
  GS_CUDA_ERROR = 8,
  GS_NO_DEVICE = 9,
  GS_PARSE_ERROR = 10,       /* ParseError{line}, core.hpp:95-100 (line: gs_last_parse_line) */
  GS_UNSUPPORTED_FORMAT = 11,/* UnsupportedFormat, core.hpp:102-104 */
  GS_IO_ERROR = 12,          /* std::runtime_error "cannot open ..." (pipeline_io.cpp:160-182) */
  GS_DEGENERATE = 13,        /* DegenerateConfiguration, core.hpp:106-108 */
  GS_INTERNAL = 99
} gs_status;

/* ConfigViolation bits (core.hpp:215-220), in declaration order. */
enum {
  GS_VIOLATION_NON_POSITIVE_SIGMA = 1u << 0,
  GS_VIOLATION_NON_POSITIVE_LAMBDA = 1u << 1,
  GS_VIOLATION_ZERO_TIMESTEPS = 1u << 2,
  GS_VIOLATION_NON_POSITIVE_THRESHOLD = 1u << 3
};

typedef enum gs_precision { GS_F64 = 0, GS_F32 = 1 } gs_precision;
typedef enum gs_backend { GS_EXACT = 0, GS_BARNES_HUT = 1 } gs_backend;
/* The reference integrates with explicit Euler only (shooting.hpp:16-18).
 * GS_RK4 is the classical four-stage scheme over the same RHS (BASELINE
 * config 4), the Barnes-Hut tree rebuilt at every stage. */
typedef enum gs_integrator { GS_EULER = 0, GS_RK4 = 1 } gs_integrator;

/* ShootingConfig (core.hpp:204-213) plus the B200 knobs. */
typedef struct gs_config {
  double sigma;                /* kernel width */
  double lambda;               /* data-attachment weight */
  int32_t timesteps;           /* uniform steps over [0, 1] */
  int32_t backend;             /* gs_backend */
  double threshold_multiplier; /* BH opening threshold = multiplier * sigma (3 by default) */
  int32_t integrator;          /* gs_integrator */
  int32_t precision;           /* gs_precision of the device arithmetic */
  /* Barnes-Hut aggregate dot scale: 0 = 1 (reference default), 1 = 1/count
   * (the reference built with GEOSHOOT_BH_LITERAL_MEAN_DOT, bh_kernel.cpp:19-26). */
  int32_t literal_mean_dot;
  uint32_t flags;              /* gs_config_flag bits (0 = reference behaviour) */
} gs_config;

/* gs_config.flags. GS_FLAG_EXACT_CUTOFF: FP32 exact flows evaluate the
 * all-pairs sum over Morton-ordered points and skip (target block, source
 * tile) pairs farther apart than the FP32 underflow radius of the Gaussian
 * (every weight there is exactly 0): bit-identical to evaluating those pairs,
 * in the same Morton order (GS_FLAG_EXACT_MORTON, the no-skip counterpart,
 * exists to test exactly that). Unsharded FP32 flows only; ignored otherwise. */
typedef enum gs_config_flag {
  GS_FLAG_EXACT_CUTOFF = 1u,
  GS_FLAG_EXACT_MORTON = 2u
} gs_config_flag;

/* Reference defaults (core.hpp:204-213): sigma 2, lambda 1, 40 steps, exact,
 * 3 sigma; Euler; F64. */
gs_config gs_default_config(void);

/* TraversalStats (bh_kernel.hpp:28-38) + EvalStats (shooting.hpp:41-55). */
typedef struct gs_stats {
  uint64_t direct_interactions;
  uint64_t approximated_interactions;
  uint64_t nodes_visited;
  uint64_t traversal_queries;
  double tree_build_ms;
  double forward_ms;
  double backward_ms;
} gs_stats;

/* ObjectiveReport (shooting.hpp:33-38). */
typedef struct gs_report {
  double energy;
  double attachment;
  double total;
  double residual_sse;
} gs_report;

typedef struct gs_ctx gs_ctx;

/* ---- context --------------------------------------------------------------- */
gs_ctx* gs_create(int device, gs_status* status);
/* Multi-device context over devices[0..count) (1 <= count <= 16) in one
 * process (replaces running the reference's parallel_for on one
 * host): one sub-context (device, stream, workspaces) per target shard, peer
 * access enabled between the distinct devices. gs_shoot_forward, gs_objective,
 * gs_evaluate, gs_optimize and the gs_flow_* calls on it shard the target
 * points into `count` contiguous ranges (Barnes-Hut: of the Morton-ordered
 * points). Every device holds all records; each stage epilogue stores its
 * shard's updated records into every peer's buffer (P2P stores over NVLink /
 * NVSwitch -- the per-stage all-gather fused into the epilogue; explicit peer
 * copies where P2P is unavailable), records ping-pong between stages and one
 * event wait per peer orders them. The adjoint pass exchanges the (alpha,
 * beta) shards the same way. Exact results are bit-identical to a
 * one-device context (shards are planned as the full problem); Barnes-Hut
 * results have the same interaction sets (summation order may differ).
 * A device may be listed more than once: its shards then run on separate
 * streams of that device (used to test the sharding on one GPU). The other
 * entry points run on devices[0]. */
gs_ctx* gs_create_multi(int32_t count, const int32_t* devices, gs_status* status);
/* Devices (shards) of a context: 1 for gs_create. */
int32_t gs_ctx_device_count(const gs_ctx* ctx);
/* 1 if the multi-device exchange uses P2P stores from the epilogues. */
int32_t gs_ctx_peer_stores(const gs_ctx* ctx);
/* Flows and trees made on the context are detached, not freed: afterwards
   they may only be released (gs_flow_destroy / gs_tree_free). */
void gs_destroy(gs_ctx* ctx);
const char* gs_last_error(const gs_ctx* ctx);
/* Literal-mean-dot mode of the context's tree-level Barnes-Hut calls
 * (gs_bh_rhs / gs_bh_hessian_products / gs_bh_hamiltonian): the reference's
 * compile-time GEOSHOOT_BH_LITERAL_MEAN_DOT switch (bh_kernel.cpp:19-26) as a
 * runtime setting. Shooting calls take it from gs_config.literal_mean_dot. */
gs_status gs_set_literal_mean_dot(gs_ctx* ctx, int32_t enable);
int gs_last_nonfinite_step(const gs_ctx* ctx);
uint32_t gs_last_config_violations(const gs_ctx* ctx);
int gs_abi_version(void);
/* Barnes-Hut walk selection, process-wide (diagnosis / parity sweeps; the
 * GS_BH_KERNEL / GS_BH_TASKS environment variables set the same defaults):
 * kernel 0 = by regime (group walk for dense near fields, else independent
 * walks), 1 = independent walks, 3 = group walk, 4 = split by warp query box;
 * windows 0 = automatic node windows, K = K windows (<= 64); -1 restores the
 * environment's choice. Every choice gives the reference's interaction sets. */
gs_status gs_set_bh_walk(int32_t kernel, int32_t windows);
/* Exact FP32 all-pairs formulation, process-wide (GS_EXACT_PAIRS sets the
 * default): 0 = by size (the symmetric kernels from 8k points; unsharded), 1 = gather
 * (each ordered pair per target, k_rhs_f32x2), 2 = symmetric whenever it
 * applies (each unordered pair once, fed to both ends, as the reference's
 * i < j sweep, kernel_exact.cpp:29-61); -1 restores the environment's choice. */
gs_status gs_set_exact_pairs(int32_t mode);
/* The formulation an unsharded exact RHS of n points takes under the current
 * choice: *tiles = T (symmetric over T tiles: 3072 / 1536 points in FP32,
 * 1024 in FP64) or 0 (gather). */
gs_status gs_exact_pairs_plan(int32_t precision, int64_t n, int32_t* tiles);
/* validate_config, core.cpp:5-17: every violated bound in *mask. */
gs_status gs_validate_config(const gs_config* cfg, uint32_t* mask);

/* ---- kernel_exact (kernel_exact.hpp:37-80) ---------------------------------- */
/* hamiltonian, kernel_exact.cpp:13-27. */
gs_status gs_hamiltonian(gs_ctx* ctx, int32_t precision, int64_t n, const double* q,
                         const double* p, double sigma, double* h_out);
/* hamiltonian_with_gradients, kernel_exact.cpp:29-61 (h_out may be NULL). */
gs_status gs_exact_rhs(gs_ctx* ctx, int32_t precision, int64_t n, const double* q,
                       const double* p, double sigma, double* dH_dp, double* dH_dq,
                       double* h_out);
/* exact_velocity, kernel_exact.cpp:70-82. */
gs_status gs_exact_velocity(gs_ctx* ctx, int32_t precision, int64_t m, const double* x,
                            int64_t n, const double* q, const double* p, double sigma,
                            double* v_out);
/* hessian_products, kernel_exact.cpp:84-135. */
gs_status gs_hessian_products(gs_ctx* ctx, int32_t precision, int64_t n, const double* q,
                              const double* p, const double* alpha, const double* beta,
                              double sigma, double* pq_alpha, double* pp_alpha,
                              double* qq_beta, double* qp_beta);

/* ---- octree (octree.hpp:17-87) ---------------------------------------------- */
/* A device-resident octree with the reference's node semantics (octree.cpp:
 * 25-117: anisotropic padded root box, midpoint subdivision, single-point
 * leaves, depth-32 buckets), built from midpoint-replay Morton keys. Nodes are
 * stored in depth-first pre-order (children 0..7); points in leaf order. */
typedef struct gs_tree gs_tree;

/* Octree::build, octree.cpp:25-40. */
gs_status gs_tree_build(gs_ctx* ctx, int32_t precision, int64_t n, const double* q,
                        const double* p, gs_tree** out);
/* Octree(cell_min, cell_max) + insert of every point in index order
 * (octree.hpp:38-51): same tree over an explicit root cell; GS_OUT_OF_BOUNDS
 * if a point lies outside it (octree.cpp:76-78). */
gs_status gs_tree_build_in_cell(gs_ctx* ctx, int32_t precision, int64_t n, const double* q,
                                const double* p, const double* cell_min, const double* cell_max,
                                gs_tree** out);
void gs_tree_free(gs_tree* tree);
int64_t gs_tree_node_count(const gs_tree* tree);
int64_t gs_tree_point_count(const gs_tree* tree);
/* Octree::accumulate_adjoints, octree.cpp:119-139. */
gs_status gs_tree_accumulate_adjoints(gs_tree* tree, const double* alpha, const double* beta);
/* Host copy of the tree for inspection (any pointer may be NULL):
 *   order[n]          point index at each leaf-order position (DFS, children 0..7)
 *   key_hi/key_lo[n]  midpoint-replay Morton keys per point index (levels 1..21 / 22..32)
 *   level[m]          node depth (root 0)
 *   parent[m]         pre-order index of the parent (-1 for the root)
 *   skip[m]           pre-order index just past the node's subtree
 *   range[2m]         [first, last] leaf-order positions of the node's points
 *   boxes[12m]        cell_min, cell_max, actual_min, actual_max (octree.hpp:23-24)
 *   sums[12m]         position_sum, momentum_sum, alpha_sum, beta_sum (:25-28)
 *   count[m]          point count (:29)                                       */
gs_status gs_tree_download(const gs_tree* tree, int32_t* order, uint64_t* key_hi,
                           uint64_t* key_lo, int32_t* level, int32_t* parent,
                           int32_t* skip, int32_t* range, double* boxes, double* sums,
                           uint32_t* count);

/* ---- bh_kernel (bh_kernel.hpp:48-99) ----------------------------------------- */
/* bh_velocity, bh_kernel.cpp:62-79, for m eval points. stats may be NULL. */
gs_status gs_bh_velocity(gs_tree* tree, int64_t m, const double* x, double sigma,
                         double threshold, double* v_out, gs_stats* stats);
/* bh_hamiltonian_gradients, bh_kernel.cpp:193-210 (queries = the tree's own points). */
gs_status gs_bh_rhs(gs_tree* tree, double sigma, double threshold, double* dH_dp,
                    double* dH_dq, gs_stats* stats);
/* Per-query (direct, approximated, visited) counts of the last query call on
 * this tree -- gs_bh_rhs, gs_bh_velocity, gs_bh_hessian_products,
 * gs_bh_point_gradients, gs_bh_point_hessian_products -- as the reference's
 * per-query TraversalStats (bh_kernel.cpp:30-58): 3*m uint64, query order.
 * Counted for every walk and node-window split (windows are folded). */
gs_status gs_bh_query_stats(const gs_tree* tree, uint64_t* per_query);
/* bh_point_gradients, bh_kernel.cpp:81-112, for m arbitrary queries
 * (x[k], px[k]) -- tree points or not -- in one device traversal. */
gs_status gs_bh_point_gradients(gs_tree* tree, int64_t m, const double* x, const double* px,
                                double sigma, double threshold, double* dH_dp, double* dH_dq,
                                gs_stats* stats);
/* bh_point_hessian_products, bh_kernel.cpp:114-160, for m arbitrary queries
 * (qi[k], pi[k], alpha_i[k], beta_i[k]). Direct terms read the per-point
 * adjoints alpha/beta (n x 3 by tree point index); approximated terms read the
 * node sums of the last gs_tree_accumulate_adjoints (zero if never annotated,
 * the reference's Node defaults). alpha = beta = NULL keeps the per-point
 * adjoints of the last annotation / call. */
gs_status gs_bh_point_hessian_products(gs_tree* tree, int64_t m, const double* qi,
                                       const double* pi, const double* alpha_i,
                                       const double* beta_i, const double* alpha,
                                       const double* beta, double sigma, double threshold,
                                       double* pq_alpha, double* pp_alpha, double* qq_beta,
                                       double* qp_beta, gs_stats* stats);
/* bh_hamiltonian, bh_kernel.cpp:162-191. */
gs_status gs_bh_hamiltonian(gs_tree* tree, double sigma, double threshold, double* h_out,
                            gs_stats* stats);
/* bh_hessian_products, bh_kernel.cpp:212-236; the tree must carry the same
 * alpha/beta via gs_tree_accumulate_adjoints. */
gs_status gs_bh_hessian_products(gs_tree* tree, const double* alpha, const double* beta,
                                 double sigma, double threshold, double* pq_alpha,
                                 double* pp_alpha, double* qq_beta, double* qp_beta,
                                 gs_stats* stats);

/* ---- shooting (shooting.hpp:57-86) ------------------------------------------- */
/* shoot_forward, shooting.cpp:244-249. traj_q/traj_p: (T+1) x n x 3, or NULL
 * to return only the final state in final_q/final_p (either may be NULL).
 * energy_out: H(q0, p0) = 1/2 <p0, dH/dp> (shooting.cpp:104-108), may be NULL. */
gs_status gs_shoot_forward(gs_ctx* ctx, const gs_config* cfg, int64_t n, const double* q0,
                           const double* p0, double* traj_q, double* traj_p,
                           double* final_q, double* final_p, double* energy_out,
                           gs_stats* stats);
/* objective, shooting.cpp:251-257. */
gs_status gs_objective(gs_ctx* ctx, const gs_config* cfg, int64_t n, const double* q0,
                       const double* p0, const double* target, gs_report* report);
/* backward_gradient, shooting.cpp:259-264; `states` snapshots (must be T+1). */
gs_status gs_backward_gradient(gs_ctx* ctx, const gs_config* cfg, int64_t n, int32_t states,
                               const double* traj_q, const double* traj_p,
                               const double* target, double* grad_out);
/* warp_points, shooting.cpp:266-300. */
gs_status gs_warp_points(gs_ctx* ctx, const gs_config* cfg, int64_t n, int32_t states,
                         const double* traj_q, const double* traj_p, int64_t m,
                         const double* x, double* y_out);
/* evaluate, shooting.cpp:302-314: fused forward (trees kept on device) +
 * report + adjoint backward. */
gs_status gs_evaluate(gs_ctx* ctx, const gs_config* cfg, int64_t n, const double* q0,
                      const double* p0, const double* target, gs_report* report,
                      double* grad_out, gs_stats* stats);

/* ---- device-resident flow (bench / batched callers) --------------------------
 * A flow keeps (q, p) resident in HBM between calls so a caller can advance it
 * without host round trips; gs_shoot_forward is upload + gs_flow_advance +
 * download. Target sharding for multi-GPU: a flow owns targets
 * [shard_begin, shard_begin + shard_count) of n and exposes its packed source
 * buffer (all n points) so the caller can all-gather shards after every
 * integrator stage (see paper_1907_04834_b200/shard.py). */
typedef struct gs_flow gs_flow;
gs_status gs_flow_create(gs_ctx* ctx, const gs_config* cfg, int64_t n, gs_flow** out);
void gs_flow_destroy(gs_flow* flow);
gs_status gs_flow_upload(gs_flow* flow, const double* q0, const double* p0);
/* Advance `steps` integrator steps (each Euler step = 1 RHS, RK4 = 4) with no
 * host synchronisation; errors surface at gs_flow_sync. */
gs_status gs_flow_advance(gs_flow* flow, int32_t steps);
gs_status gs_flow_sync(gs_flow* flow);
gs_status gs_flow_download(gs_flow* flow, double* q, double* p);
/* Number of kernels the last gs_flow_advance launched (bench evidence). */
int64_t gs_flow_last_launches(const gs_flow* flow);
/* cudaStream_t of the flow (as void*), for event timing on the launch stream. */
void* gs_flow_stream(const gs_flow* flow);
/* Work counters accumulated since the last upload (TraversalStats,
 * bh_kernel.hpp:28-38): direct / approximated interactions and visited nodes
 * (Barnes-Hut, counted on the device) or ordered pairs (exact). Synchronises. */
gs_status gs_flow_stats(gs_flow* flow, gs_stats* out);

/* Event timing of the dominant kernels of subsequent advances / stages
 * (the all-pairs RHS kernel or the Barnes-Hut traversal; and the tree build),
 * on the flow's stream: summed milliseconds and launch counts since the last
 * read. */
gs_status gs_flow_profile(gs_flow* flow, int32_t enable);
gs_status gs_flow_profile_read(gs_flow* flow, double* kernel_ms, int64_t* kernel_launches,
                               double* build_ms, int64_t* builds);

/* Per-channel form of gs_flow_profile_read: channel 0 dominant kernel,
 * 1 tree build, 2..5 tree-build phases (bbox+keys, radix sort, topology,
 * aggregates); ms[c] summed, counts[c] pairs recorded. */
gs_status gs_flow_profile_phases(gs_flow* flow, double* ms, int64_t* counts, int32_t channels);

/* Event timing inside the context's shooting calls (gs_shoot_forward,
 * gs_evaluate, gs_optimize): channels as gs_flow_profile_phases, plus
 * 6 = the adjoint pass's dominant kernel (Hessian products / Barnes-Hut
 * Hessian walk). gs_profile_phases drains: ms[c] summed, counts[c] pairs. */
gs_status gs_profile(gs_ctx* ctx, int32_t enable);
gs_status gs_profile_phases(gs_ctx* ctx, double* ms, int64_t* counts, int32_t channels);

/* Kernel start-time trace (profiling; valid inside captured CUDA graphs,
 * where host events cannot look): while enabled, every traced kernel of the
 * tree build, the Barnes-Hut walks and the epilogues appends {tag, device
 * %globaltimer ns} when its first CTA starts; tag = unit << 16 | source line
 * (unit 1 tree.cu, 2 bh.cu, 3 epilogue.cu). gs_trace_read copies up to max
 * entries, returns their number in *count and clears the trace. One trace per
 * process, on the context's (first) device; entries beyond 16384 are dropped. */
gs_status gs_trace(gs_ctx* ctx, int32_t enable);
gs_status gs_trace_read(gs_ctx* ctx, uint64_t* tags, uint64_t* times_ns, int64_t max,
                        int64_t* count);

/* Sharded stage API (one rank = one flow): */
gs_status gs_flow_set_shard(gs_flow* flow, int64_t shard_begin, int64_t shard_count);
/* Device pointer and byte size of the packed per-point source records
 * (n records, record bytes = gs_flow_record_bytes); the shard's records are
 * contiguous at shard_begin. */
void* gs_flow_source_buffer(gs_flow* flow);
int64_t gs_flow_record_bytes(const gs_flow* flow);
/* One integrator stage on the shard (RHS over all n sources + fused stage
 * epilogue that rewrites the shard's records); stage = 0..stages-1 of the
 * current step (Euler 1, RK4 4). */
gs_status gs_flow_stage(gs_flow* flow, int32_t stage);
/* Multi-GPU symmetric exact stages (exact FP32 flows whose
 * problem takes the symmetric kernel, gs_exact_pairs_plan): rank `rank` of
 * `world` evaluates the unordered tile pairs of its rows of the tile-pair
 * grid -- each pair once, for both ends, as the reference's i < j sweep
 * (kernel_exact.cpp:29-61) -- instead of the gather form over its target
 * shard. *enabled = 0 when the flow does not qualify (the caller then uses
 * gs_flow_stage). A stage is then: gs_flow_stage_pairs (this rank's rows,
 * folded per target into n x 2 float4 partials {A = sum g p, B = sum c d'} on
 * the flow's stream; *partials = that device buffer), an exchange by the
 * caller (every rank sends each shard's slice to its owner), and
 * gs_flow_stage_apply (the shard's stage epilogue over nparts partials laid
 * out [part][shard_count] x 2 float4, folded in order). */
gs_status gs_flow_set_pair_rows(gs_flow* flow, int32_t rank, int32_t world, int32_t* enabled);
gs_status gs_flow_stage_pairs(gs_flow* flow, int32_t stage, void** partials);
gs_status gs_flow_stage_apply(gs_flow* flow, int32_t stage, const void* partials, int32_t nparts);

/* ---- registration optimizer ------------------------------
 * optimize(), optimizer.cpp:301-351: L-BFGS + strong-Wolfe line search over p0
 * from p0 = 0, every objective/gradient one gs_evaluate on the device.
 * OptimizerConfig + LineSearchConfig (core.hpp:190-202). */
typedef struct gs_opt_config {
  int32_t max_iterations;             /* 200 */
  int32_t memory;                     /* 10 history pairs */
  double gradient_tolerance;          /* 1e-6 (inf-norm) */
  double relative_objective_tolerance;/* 1e-9 */
  double sufficient_decrease;         /* Wolfe c1 = 1e-4 */
  double curvature;                   /* Wolfe c2 = 0.9 (strong) */
  int32_t max_trials;                 /* 20 evaluations per line search */
} gs_opt_config;
/* TerminationReason (optimizer.hpp:18-24), in declaration order. */
enum {
  GS_TERM_GRADIENT_TOLERANCE = 0,
  GS_TERM_OBJECTIVE_TOLERANCE = 1,
  GS_TERM_MAX_ITERATIONS = 2,
  GS_TERM_LINE_SEARCH_FAILURE = 3,
  GS_TERM_NON_FINITE = 4
};
gs_opt_config gs_default_opt_config(void);
/* p_out: n x 3 optimal momenta. trace (optional): up to max_iterations + 1
 * rows of {iter, total, energy, attachment, grad_inf, wall_ms} (the
 * reference's trace CSV columns, optimizer.cpp:204-213); GS_NONFINITE if the
 * objective is non-finite at p0 = 0 (NonFiniteObjectiveAtStart). */
gs_status gs_optimize(gs_ctx* ctx, const gs_config* cfg, const gs_opt_config* opt, int64_t n,
                      const double* q0, const double* target, double* p_out, int32_t* reason,
                      int32_t* iterations, int32_t* evaluations, double* trace,
                      int32_t* trace_len, gs_stats* stats);

/* Batched independent registrations (BASELINE config 5, "replicas only"):
 * subject b has n[b] points; each runs gs_optimize on its own context/stream
 * and host thread so the device overlaps them. final_total[b] = objective at
 * the returned p0. */
gs_status gs_optimize_batch(int device, const gs_config* cfg, const gs_opt_config* opt,
                            int32_t batch, const int64_t* n, const double* const* q0,
                            const double* const* target, double* const* p_out, int32_t* reasons,
                            int32_t* iterations, int32_t* evaluations, double* final_total);

/* Batched independent evaluations (SURVEY.md §8b gs_evaluate_batch): subject b
 * (n[b] points, its own q0 / p0 / target) runs gs_evaluate on its own
 * context/stream and host thread; reports[b], grad_out[b] (n[b] x 3) and
 * stats[b] (optional) as gs_evaluate. Results equal one-at-a-time calls. */
gs_status gs_evaluate_batch(int device, const gs_config* cfg, int32_t batch, const int64_t* n,
                            const double* const* q0, const double* const* p0,
                            const double* const* target, gs_report* reports,
                            double* const* grad_out, gs_stats* stats);

/* ---- point-cloud files (pipeline.hpp:52-68) ---------------
 * xyz text ("x y z" per line, '#' comments) and legacy-VTK ASCII polydata
 * (points only); output with %.17g, so values round-trip bit-exactly. */
typedef enum gs_point_format { GS_FORMAT_XYZ = 0, GS_FORMAT_VTK = 1 } gs_point_format;
/* format_for_path, pipeline_io.cpp:153-158: ".vtk" -> VTK, else xyz. */
int32_t gs_format_for_path(const char* path);
/* read_points: call with xyz_out = NULL to get *n_out, then with capacity >= n. */
gs_status gs_read_points(const char* path, int32_t format, double* xyz_out, int64_t capacity,
                         int64_t* n_out);
/* write_points: header lines become '#' comments (xyz) or the title (VTK). */
gs_status gs_write_points(const char* path, int32_t format, int64_t n, const double* xyz,
                          const char* const* header, int32_t n_header);
long long gs_last_parse_line(void);
const char* gs_last_io_error(void);

/* ---- rigid pre-alignment (procrustes.cpp:7-58) -----------
 * Least-squares rotation + translation taking source onto target (index
 * correspondence, reflection-corrected). Centroids, cross-covariance and the
 * transform of every point on the device (FP64); the 3x3 SVD on the host.
 * rotation_rows[9] row-major, translation[3], aligned_out n x 3 (any may be
 * NULL). GS_DEGENERATE for n < 3 or collinear sources. */
gs_status gs_procrustes_align(gs_ctx* ctx, int64_t n, const double* source, const double* target,
                              double* rotation_rows, double* translation, double* aligned_out);

/* ---- measured device peaks (roofline denominators) ----------------------------
 * kind 0: FP32 FFMA lane-ops/s (constant operands), 1: MUFU.EX2 lane-ops/s,
 * 2: FP64 DFMA lane-ops/s, 3: FP32 FFMA lane-ops/s with all-register operands,
 * 4: FP32 lane-FMAs/s issued as packed FFMA2 (2 per lane per instruction). */
gs_status gs_microbench(int device, int32_t kind, double* ops_per_s);

#ifdef __cplusplus
}
#endif
#endif /* GEOSHOOT_B200_H */
