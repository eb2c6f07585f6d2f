// TEST INFRASTRUCTURE ONLY -- never linked into, or called by, the product.
//
// Plain-array C shim over the UNMODIFIED reference sources, which
// oracle/Makefile compiles by path from $(GEOSHOOT_REF_DIR)/src into
// oracle/_ref/libgeoshoot_ref.so (namespace renamed to geoshoot_ref so it can
// never collide with the product's C++ API). Only tests/, __graft_entry__.smoke()
// and bench.py's reference / cpu_baseline legs load it, as the checker.
//
// Every entry point forwards to the reference function named in its comment
// (file:line under /root/reference/proj) with no arithmetic of its own, except
// ref_bh_rhs / ref_bh_hessprod, which replay the per-point parallel_for loops
// of shooting.cpp:136-142 and :278-286 over the reference per-point kernels.
//
// Status codes match include/geoshoot_b200.h (gs_status).

#include <cstdint>
#include <cstring>
#include <exception>
#include <thread>
#include <vector>

#include "geoshoot/bh_kernel.hpp"
#include "geoshoot/core.hpp"
#include "geoshoot/kernel_exact.hpp"
#include "geoshoot/octree.hpp"
#include "geoshoot/optimizer.hpp"
#include "geoshoot/parallel.hpp"
#include "geoshoot/pipeline.hpp"
#include "geoshoot/shooting.hpp"
#include "geoshoot/synthetic.hpp"

using namespace geoshoot;  // renamed by -Dgeoshoot=geoshoot_ref[_lmd] (oracle/Makefile)

namespace {

enum : int {
  kOk = 0,
  kDimensionMismatch = 1,
  kConfigError = 2,
  kNonFinite = 3,
  kConfigMismatch = 4,
  kEmptyTree = 5,
  kOutOfBounds = 6,
  kInvalidArgument = 7,
  kInternal = 99,
};

std::vector<Vec3> vecs(const double* xyz, std::int64_t n) {
  std::vector<Vec3> v(static_cast<std::size_t>(n));
  if (n > 0) std::memcpy(v.data(), xyz, sizeof(double) * 3 * n);
  return v;
}

void store(double* out, const std::vector<Vec3>& v) {
  if (out && !v.empty()) std::memcpy(out, v.data(), sizeof(double) * 3 * v.size());
}

ShootingConfig make_cfg(double sigma, double lambda, int timesteps, int backend,
                        double thr_mult) {
  ShootingConfig c;
  c.sigma = sigma;
  c.lambda = lambda;
  c.timesteps = timesteps;
  c.backend = backend ? Backend::BarnesHut : Backend::Exact;
  c.threshold_multiplier = thr_mult;
  return c;
}

thread_local int g_nonfinite_step = 0;
thread_local std::uint32_t g_config_mask = 0;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const NonFiniteState& e) {
    g_nonfinite_step = e.timestep;
    return kNonFinite;
  } catch (const ConfigError& e) {
    g_config_mask = 0;
    for (ConfigViolation v : e.violations) g_config_mask |= 1u << static_cast<int>(v);
    return kConfigError;
  } catch (const DimensionMismatch&) {
    return kDimensionMismatch;
  } catch (const ConfigMismatch&) {
    return kConfigMismatch;
  } catch (const EmptyTree&) {
    return kEmptyTree;
  } catch (const OutOfBounds&) {
    return kOutOfBounds;
  } catch (const std::invalid_argument&) {
    return kInvalidArgument;
  } catch (...) {
    return kInternal;
  }
}

}  // namespace

extern "C" {

int ref_last_nonfinite_step() { return g_nonfinite_step; }
unsigned ref_last_config_mask() { return g_config_mask; }

// kernel_exact.cpp:13-27
int ref_hamiltonian(std::int64_t n, const double* q, const double* p, double sigma,
                    double* h_out) {
  return guarded([&] {
    *h_out = hamiltonian(PointSet(vecs(q, n)), MomentumSet(vecs(p, n)), sigma);
  });
}

// kernel_exact.cpp:29-61 (hamiltonian_with_gradients)
int ref_exact_rhs(std::int64_t n, const double* q, const double* p, double sigma,
                  double* dHdp, double* dHdq, double* h_out) {
  return guarded([&] {
    HamiltonianGradients g;
    const double h =
        hamiltonian_with_gradients(PointSet(vecs(q, n)), MomentumSet(vecs(p, n)), sigma, g);
    store(dHdp, g.dH_dp);
    store(dHdq, g.dH_dq);
    if (h_out) *h_out = h;
  });
}

// Runs hamiltonian_gradients (kernel_exact.cpp:63-68) `reps` times on each of
// `threads` host threads concurrently (independent calls; the reference exact
// path is serial by construction, kernel_exact.cpp:29-61). Used only by the
// CPU baseline to occupy every host core with the reference's own RHS.
int ref_exact_rhs_concurrent(std::int64_t n, const double* q, const double* p,
                             double sigma, int threads, int reps, double* dHdp,
                             double* dHdq) {
  return guarded([&] {
    const PointSet qs(vecs(q, n));
    const MomentumSet ps(vecs(p, n));
    std::vector<HamiltonianGradients> outs(static_cast<std::size_t>(threads));
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        for (int r = 0; r < reps; ++r) outs[t] = hamiltonian_gradients(qs, ps, sigma);
      });
    for (auto& th : pool) th.join();
    store(dHdp, outs[0].dH_dp);
    store(dHdq, outs[0].dH_dq);
  });
}

// kernel_exact.cpp:70-82
int ref_exact_velocity(std::int64_t m, const double* x, std::int64_t n, const double* q,
                       const double* p, double sigma, double* v_out) {
  return guarded([&] {
    store(v_out, exact_velocity(PointSet(vecs(x, m)), PointSet(vecs(q, n)),
                                MomentumSet(vecs(p, n)), sigma));
  });
}

// kernel_exact.cpp:84-135
int ref_hessian_products(std::int64_t n, const double* q, const double* p,
                         const double* alpha, const double* beta, double sigma,
                         double* pq, double* pp, double* qq, double* qp) {
  return guarded([&] {
    const HessianProducts h = hessian_products(PointSet(vecs(q, n)), MomentumSet(vecs(p, n)),
                                               vecs(alpha, n), vecs(beta, n), sigma);
    store(pq, h.pq_alpha);
    store(pp, h.pp_alpha);
    store(qq, h.qq_beta);
    store(qp, h.qp_beta);
  });
}

// ---------------------------------------------------------------- octree ---

// Octree::build, octree.cpp:25-40. Returns an owning handle.
void* ref_tree_build(std::int64_t n, const double* q, const double* p, int* status) {
  Octree* t = nullptr;
  *status = guarded([&] {
    t = new Octree(Octree::build(PointSet(vecs(q, n)), MomentumSet(vecs(p, n))));
  });
  return t;
}

void ref_tree_free(void* h) { delete static_cast<Octree*>(h); }

std::int64_t ref_tree_node_count(void* h) {
  return static_cast<std::int64_t>(static_cast<Octree*>(h)->node_count());
}

// Dumps every node (octree.hpp:22-36) into flat arrays, node order as stored.
// boxes: n_nodes x 12 doubles (cell_min, cell_max, actual_min, actual_max)
// sums:  n_nodes x 12 doubles (position_sum, momentum_sum, alpha_sum, beta_sum)
// ints:  n_nodes x 11 int32   (count, children[8], first_point, leaf)
void ref_tree_dump(void* h, double* boxes, double* sums, std::int32_t* ints,
                   std::int32_t* next_point) {
  const Octree& t = *static_cast<Octree*>(h);
  for (std::size_t k = 0; k < t.node_count(); ++k) {
    const Octree::Node& nd = t.node(k);
    const Vec3 b[4] = {nd.cell_min, nd.cell_max, nd.actual_min, nd.actual_max};
    const Vec3 s[4] = {nd.position_sum, nd.momentum_sum, nd.alpha_sum, nd.beta_sum};
    std::memcpy(boxes + 12 * k, b, sizeof b);
    std::memcpy(sums + 12 * k, s, sizeof s);
    std::int32_t* o = ints + 11 * k;
    o[0] = static_cast<std::int32_t>(nd.count);
    for (int c = 0; c < 8; ++c) o[1 + c] = nd.children[c];
    o[9] = nd.first_point;
    o[10] = nd.leaf ? 1 : 0;
  }
  const auto& nx = t.next_point();
  for (std::size_t i = 0; i < nx.size(); ++i) next_point[i] = nx[i];
}

// Octree::accumulate_adjoints, octree.cpp:119-139
int ref_tree_accumulate(void* h, std::int64_t n, const double* alpha, const double* beta) {
  return guarded([&] {
    static_cast<Octree*>(h)->accumulate_adjoints(vecs(alpha, n), vecs(beta, n));
  });
}

// ------------------------------------------------------------- bh_kernel ---

// bh_velocity, bh_kernel.cpp:62-79, per eval point; stats[3] summed.
int ref_bh_velocity(void* h, std::int64_t m, const double* x, double sigma, double thr,
                    double* v_out, std::uint64_t* stats) {
  return guarded([&] {
    const Octree& t = *static_cast<Octree*>(h);
    TraversalStats acc;
    for (std::int64_t e = 0; e < m; ++e) {
      const BhVelocity r = bh_velocity(t, Vec3{x[3 * e], x[3 * e + 1], x[3 * e + 2]}, sigma, thr);
      v_out[3 * e] = r.velocity.x;
      v_out[3 * e + 1] = r.velocity.y;
      v_out[3 * e + 2] = r.velocity.z;
      acc.merge(r.stats);
    }
    if (stats) {
      stats[0] = acc.direct_interactions;
      stats[1] = acc.approximated_interactions;
      stats[2] = acc.nodes_visited;
    }
  });
}

// bh_point_gradients (bh_kernel.cpp:81-112) over every point, threaded the way
// step_gradients does it (shooting.cpp:136-142). per_query: optional n x 3
// u64 (direct, approx, visited) per query.
int ref_bh_rhs(void* h, std::int64_t n, const double* q, const double* p, double sigma,
               double thr, int threads, double* dHdp, double* dHdq, std::uint64_t* per_query) {
  return guarded([&] {
    const Octree& t = *static_cast<Octree*>(h);
    require_aligned(static_cast<std::size_t>(n), t.point_count(), "ref_bh_rhs");
    const std::vector<Vec3> qs = vecs(q, n), ps = vecs(p, n);
    const int th = threads > 0 ? threads : default_thread_count();
    parallel_for(static_cast<std::size_t>(n), th, [&](std::size_t i) {
      TraversalStats st;
      const BhPointGradients g = bh_point_gradients(t, qs[i], ps[i], sigma, thr, &st);
      std::memcpy(dHdp + 3 * i, &g.dH_dp, sizeof(Vec3));
      std::memcpy(dHdq + 3 * i, &g.dH_dq, sizeof(Vec3));
      if (per_query) {
        per_query[3 * i] = st.direct_interactions;
        per_query[3 * i + 1] = st.approximated_interactions;
        per_query[3 * i + 2] = st.nodes_visited;
      }
    });
  });
}

// bh_point_hessian_products (bh_kernel.cpp:114-160) over every point, threaded
// as run_backward does (shooting.cpp:278-286). The tree must already carry
// accumulate_adjoints(alpha, beta).
int ref_bh_hessprod(void* h, std::int64_t n, const double* q, const double* p,
                    const double* alpha, const double* beta, double sigma, double thr,
                    int threads, double* pq, double* pp, double* qq, double* qp,
                    std::uint64_t* per_query) {
  return guarded([&] {
    const Octree& t = *static_cast<Octree*>(h);
    const std::vector<Vec3> qs = vecs(q, n), ps = vecs(p, n), as = vecs(alpha, n),
                            bs = vecs(beta, n);
    const int th = threads > 0 ? threads : default_thread_count();
    parallel_for(static_cast<std::size_t>(n), th, [&](std::size_t i) {
      TraversalStats st;
      const BhPointHessianProducts r = bh_point_hessian_products(
          t, qs[i], ps[i], as[i], bs[i], as, bs, sigma, thr, &st);
      std::memcpy(pq + 3 * i, &r.pq_alpha, sizeof(Vec3));
      std::memcpy(pp + 3 * i, &r.pp_alpha, sizeof(Vec3));
      std::memcpy(qq + 3 * i, &r.qq_beta, sizeof(Vec3));
      std::memcpy(qp + 3 * i, &r.qp_beta, sizeof(Vec3));
      if (per_query) {
        per_query[3 * i] = st.direct_interactions;
        per_query[3 * i + 1] = st.approximated_interactions;
        per_query[3 * i + 2] = st.nodes_visited;
      }
    });
  });
}

// bh_point_gradients (bh_kernel.cpp:81-112) at m arbitrary queries (x, px);
// per_query: optional m x 3 (direct, approx, visited).
int ref_bh_point_gradients(void* h, std::int64_t m, const double* x, const double* px,
                           double sigma, double thr, int threads, double* dHdp, double* dHdq,
                           std::uint64_t* per_query) {
  return guarded([&] {
    const Octree& t = *static_cast<Octree*>(h);
    const std::vector<Vec3> xs = vecs(x, m), ps = vecs(px, m);
    const int th = threads > 0 ? threads : default_thread_count();
    parallel_for(static_cast<std::size_t>(m), th, [&](std::size_t i) {
      TraversalStats st;
      const BhPointGradients g = bh_point_gradients(t, xs[i], ps[i], sigma, thr, &st);
      std::memcpy(dHdp + 3 * i, &g.dH_dp, sizeof(Vec3));
      std::memcpy(dHdq + 3 * i, &g.dH_dq, sizeof(Vec3));
      if (per_query) {
        per_query[3 * i] = st.direct_interactions;
        per_query[3 * i + 1] = st.approximated_interactions;
        per_query[3 * i + 2] = st.nodes_visited;
      }
    });
  });
}

// bh_point_hessian_products (bh_kernel.cpp:114-160) at m arbitrary queries
// (qi, pi, alpha_i, beta_i); alpha/beta (n x 3) are the direct terms' per-point
// adjoints; the tree's node sums are whatever accumulate_adjoints left.
int ref_bh_point_hessprod(void* h, std::int64_t m, const double* qi, const double* pi,
                          const double* ai, const double* bi, std::int64_t n, const double* alpha,
                          const double* beta, double sigma, double thr, int threads, double* pq,
                          double* pp, double* qq, double* qp, std::uint64_t* per_query) {
  return guarded([&] {
    const Octree& t = *static_cast<Octree*>(h);
    const std::vector<Vec3> qs = vecs(qi, m), ps = vecs(pi, m), as_i = vecs(ai, m),
                            bs_i = vecs(bi, m), as = vecs(alpha, n), bs = vecs(beta, n);
    const int th = threads > 0 ? threads : default_thread_count();
    parallel_for(static_cast<std::size_t>(m), th, [&](std::size_t i) {
      TraversalStats st;
      const BhPointHessianProducts r = bh_point_hessian_products(
          t, qs[i], ps[i], as_i[i], bs_i[i], as, bs, sigma, thr, &st);
      std::memcpy(pq + 3 * i, &r.pq_alpha, sizeof(Vec3));
      std::memcpy(pp + 3 * i, &r.pp_alpha, sizeof(Vec3));
      std::memcpy(qq + 3 * i, &r.qq_beta, sizeof(Vec3));
      std::memcpy(qp + 3 * i, &r.qp_beta, sizeof(Vec3));
      if (per_query) {
        per_query[3 * i] = st.direct_interactions;
        per_query[3 * i + 1] = st.approximated_interactions;
        per_query[3 * i + 2] = st.nodes_visited;
      }
    });
  });
}

// bh_velocity (bh_kernel.cpp:62-79) per eval point with per-query stats, threaded.
int ref_bh_velocity_pq(void* h, std::int64_t m, const double* x, double sigma, double thr,
                       int threads, double* v_out, std::uint64_t* per_query) {
  return guarded([&] {
    const Octree& t = *static_cast<Octree*>(h);
    const int th = threads > 0 ? threads : default_thread_count();
    parallel_for(static_cast<std::size_t>(m), th, [&](std::size_t e) {
      const BhVelocity r = bh_velocity(t, Vec3{x[3 * e], x[3 * e + 1], x[3 * e + 2]}, sigma, thr);
      std::memcpy(v_out + 3 * e, &r.velocity, sizeof(Vec3));
      per_query[3 * e] = r.stats.direct_interactions;
      per_query[3 * e + 1] = r.stats.approximated_interactions;
      per_query[3 * e + 2] = r.stats.nodes_visited;
    });
  });
}

// bh_hamiltonian, bh_kernel.cpp:162-191
int ref_bh_hamiltonian(void* h, std::int64_t n, const double* q, const double* p,
                       double sigma, double thr, double* h_out) {
  return guarded([&] {
    *h_out = bh_hamiltonian(*static_cast<Octree*>(h), PointSet(vecs(q, n)),
                            MomentumSet(vecs(p, n)), sigma, thr, nullptr);
  });
}

// -------------------------------------------------------------- shooting ---

// shoot_forward, shooting.cpp:244-249. traj_q/traj_p: (T+1) x n x 3.
int ref_shoot_forward(std::int64_t n, const double* q0, const double* p0, double sigma,
                      int timesteps, int backend, double thr_mult, double* traj_q,
                      double* traj_p) {
  return guarded([&] {
    const GeodesicTrajectory tr =
        shoot_forward(PointSet(vecs(q0, n)), MomentumSet(vecs(p0, n)),
                      make_cfg(sigma, 1.0, timesteps, backend, thr_mult));
    for (std::size_t k = 0; k < tr.states.size(); ++k) {
      store(traj_q + k * 3 * n, tr.states[k].q.data());
      store(traj_p + k * 3 * n, tr.states[k].p.data());
    }
  });
}

// objective, shooting.cpp:251-257. report: energy, attachment, total, sse.
int ref_objective(std::int64_t n, const double* q0, const double* p0, const double* target,
                  double sigma, double lambda, int timesteps, int backend, double thr_mult,
                  double* report) {
  return guarded([&] {
    const ObjectiveReport r =
        objective(PointSet(vecs(q0, n)), MomentumSet(vecs(p0, n)), PointSet(vecs(target, n)),
                  make_cfg(sigma, lambda, timesteps, backend, thr_mult));
    report[0] = r.energy;
    report[1] = r.attachment;
    report[2] = r.total;
    report[3] = r.residual_sse;
  });
}

// evaluate, shooting.cpp:302-314. stats: direct, approx, visited, queries.
int ref_evaluate(std::int64_t n, const double* q0, const double* p0, const double* target,
                 double sigma, double lambda, int timesteps, int backend, double thr_mult,
                 int threads, double* report, double* grad, std::uint64_t* stats,
                 double* times_ms) {
  return guarded([&] {
    const Evaluation ev =
        evaluate(PointSet(vecs(q0, n)), MomentumSet(vecs(p0, n)), PointSet(vecs(target, n)),
                 make_cfg(sigma, lambda, timesteps, backend, thr_mult), threads);
    report[0] = ev.report.energy;
    report[1] = ev.report.attachment;
    report[2] = ev.report.total;
    report[3] = ev.report.residual_sse;
    store(grad, ev.gradient);
    if (stats) {
      stats[0] = ev.stats.traversal.direct_interactions;
      stats[1] = ev.stats.traversal.approximated_interactions;
      stats[2] = ev.stats.traversal.nodes_visited;
      stats[3] = ev.stats.traversal_queries;
    }
    if (times_ms) {
      times_ms[0] = ev.stats.tree_build_ms;
      times_ms[1] = ev.stats.forward_ms;
      times_ms[2] = ev.stats.backward_ms;
    }
  });
}

static GeodesicTrajectory make_traj(std::int64_t n, int timesteps, const double* traj_q,
                                    const double* traj_p) {
  GeodesicTrajectory tr;
  for (int k = 0; k <= timesteps; ++k)
    tr.states.push_back({PointSet(vecs(traj_q + k * 3 * n, n)),
                         MomentumSet(vecs(traj_p + k * 3 * n, n))});
  return tr;
}

// backward_gradient, shooting.cpp:259-264. The trajectory has `states` snapshots.
int ref_backward_gradient(std::int64_t n, int states, const double* traj_q,
                          const double* traj_p, const double* target, double sigma,
                          double lambda, int timesteps, int backend, double thr_mult,
                          double* grad) {
  return guarded([&] {
    store(grad, backward_gradient(make_traj(n, states - 1, traj_q, traj_p),
                                  PointSet(vecs(target, n)),
                                  make_cfg(sigma, lambda, timesteps, backend, thr_mult)));
  });
}

// warp_points, shooting.cpp:266-300
int ref_warp_points(std::int64_t n, int states, const double* traj_q, const double* traj_p,
                    std::int64_t m, const double* x, double sigma, int timesteps, int backend,
                    double thr_mult, double* y_out) {
  return guarded([&] {
    const PointSet y = warp_points(make_traj(n, states - 1, traj_q, traj_p),
                                   PointSet(vecs(x, m)),
                                   make_cfg(sigma, 1.0, timesteps, backend, thr_mult));
    store(y_out, y.data());
  });
}

// optimize, optimizer.cpp:301-351 (threads = 0: process default)
int ref_optimize(std::int64_t n, const double* q0, const double* target, double sigma,
                 double lambda, int timesteps, int backend, double thr_mult, int max_iterations,
                 double* p_out, int* reason, int* iterations, double* trace, int* trace_len) {
  return guarded([&] {
    ShootingConfig c = make_cfg(sigma, lambda, timesteps, backend, thr_mult);
    c.optimizer.max_iterations = max_iterations;
    auto [p, tr] = optimize(PointSet(vecs(q0, n)), PointSet(vecs(target, n)), c, nullptr, 0);
    store(p_out, p.data());
    *reason = static_cast<int>(tr.reason);
    *iterations = tr.records.empty() ? 0 : tr.records.back().iteration;
    for (std::size_t k = 0; k < tr.records.size(); ++k) {
      const auto& r = tr.records[k];
      double* o = trace + 6 * k;
      o[0] = r.iteration; o[1] = r.total; o[2] = r.energy; o[3] = r.attachment;
      o[4] = r.grad_inf; o[5] = r.wall_ms;
    }
    *trace_len = static_cast<int>(tr.records.size());
  });
}

// read_points / write_points, pipeline_io.cpp:160-182. status 10 = ParseError
// (line in *line), 11 = UnsupportedFormat, 12 = runtime_error (open failure).
int ref_read_points(const char* path, int vtk, double* out, std::int64_t cap, std::int64_t* n,
                    long long* line) {
  try {
    const PointSet p = read_points(path, vtk ? PointFormat::LegacyPolydataAscii : PointFormat::XyzText);
    *n = static_cast<std::int64_t>(p.size());
    if (out && cap >= *n) store(out, p.data());
    return kOk;
  } catch (const ParseError& e) {
    *line = static_cast<long long>(e.line);
    return 10;
  } catch (const UnsupportedFormat&) {
    return 11;
  } catch (const std::invalid_argument&) {
    return kInvalidArgument;
  } catch (const std::runtime_error&) {
    return 12;
  }
}

int ref_write_points(const char* path, int vtk, std::int64_t n, const double* xyz,
                     const char* header) {
  return guarded([&] {
    std::vector<std::string> h;
    if (header) h.push_back(header);
    write_points(PointSet(vecs(xyz, n)), path,
                 vtk ? PointFormat::LegacyPolydataAscii : PointFormat::XyzText, h);
  });
}

// validate_config, core.cpp:5-17 -> violation bitmask (0 = valid)
unsigned ref_validate_config(double sigma, double lambda, int timesteps, double thr_mult) {
  g_config_mask = 0;
  const int st = guarded([&] { validate_config(make_cfg(sigma, lambda, timesteps, 0, thr_mult)); });
  return st == kOk ? 0u : g_config_mask;
}

// synthetic.cpp generate(): fixture shapes used by the reference tests.
// kind: 0 circle(n, a), 1 flat_rectangle(n, a=length, b=width),
// 2 bent_rectangle(n, angle=c, a, b), 3 uniform_box(n, a=extent, seed),
// 4 clustered_pairs(n, a=extent, b=spread, seed)
int ref_generate(int kind, int n, double a, double b, double c, std::uint64_t seed,
                 double* out) {
  return guarded([&] {
    ShapeSpec s;
    switch (kind) {
      case 0: s = ShapeSpec::circle(n, a); break;
      case 1: s = ShapeSpec::flat_rectangle(n, a, b); break;
      case 2: s = ShapeSpec::bent_rectangle(n, c, a, b); break;
      case 3: s = ShapeSpec::uniform_box(n, a, seed); break;
      default: s = ShapeSpec::clustered_pairs(n, a, b, seed); break;
    }
    store(out, generate(s).data());
  });
}

}  // extern "C"
