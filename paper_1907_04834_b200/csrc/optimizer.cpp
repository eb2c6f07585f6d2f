// optimizer.cpp -- the registration optimizer as a
// caller of the device evaluate(): limited-memory BFGS with a strong-Wolfe
// line search over the initial momenta, starting from p0 = 0.
//
// Restates the reference's algorithm (proj/src/optimizer.cpp): two-loop
// recursion with gamma = s.y / y.y scaling (:37-58), steepest-descent restart
// on a non-descent direction (:243-247), initial step 1/max(1, |g|_inf) on an
// empty history (:248-249), bracketing by doubling then bisection zoom within
// a shared trial budget, falling back to the best sufficient-decrease point
// (:82-189), curvature-gated history updates (:271-277) and the same
// termination order (:235-298). Non-finite flows map to +inf (:328-332).
//
// Every objective/gradient is one evaluate(): the forward flow, trees,
// adjoint and gradient run on the B200. On a single-device context the whole
// search state is device-resident too (lbfgs_dev.cu: q0 / target uploaded
// once, the O(N m) two-loop and line-search vector algebra as device kernels,
// only the steering scalars on the host); on a multi-device context the
// vectors stay on the host (below). Either way the control flow of the search
// is the reference's given the same evaluations.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <deque>
#include <limits>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "engine.h"
#include "geoshoot_b200.h"
#include "lbfgs.h"

namespace gsb {
void set_bh_concurrency(int c);  // bh.cu: flows sharing the GPU from other host threads
}

namespace {

// Contexts for the batched entry points, kept for the life of the process: a
// context owns a stream and grown device buffers, so creating and destroying
// one per subject per call (cudaFree synchronises the device) would cost more
// than the evaluation itself.
struct CtxPool {
  std::mutex mu;
  std::vector<std::pair<int, gs_ctx*>> idle;
  gs_ctx* acquire(int device, gs_status* st) {
    {
      std::lock_guard<std::mutex> g(mu);
      for (std::size_t k = 0; k < idle.size(); ++k)
        if (idle[k].first == device) {
          gs_ctx* c = idle[k].second;
          idle.erase(idle.begin() + (std::ptrdiff_t)k);
          return c;
        }
    }
    return gs_create(device, st);
  }
  void release(int device, gs_ctx* c) {
    std::lock_guard<std::mutex> g(mu);
    idle.emplace_back(device, c);
  }
};
CtxPool& ctx_pool() {
  static CtxPool* p = new CtxPool;  // never destroyed: outlives static teardown order
  return *p;
}

using Vec = std::vector<double>;
constexpr double kInf = std::numeric_limits<double>::infinity();

double vdot(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

double vmax_abs(const Vec& a) {
  double m = 0.0;
  for (double v : a) m = std::max(m, std::abs(v));
  return m;
}

struct Pair {
  Vec s, y;
  double rho;
};

// H_k g through the two-loop recursion, negated: the search direction.
Vec direction(const Vec& g, const std::deque<Pair>& hist) {
  Vec d = g;
  if (!hist.empty()) {
    std::vector<double> alpha(hist.size());
    for (std::size_t i = hist.size(); i-- > 0;) {
      alpha[i] = hist[i].rho * vdot(hist[i].s, d);
      for (std::size_t k = 0; k < d.size(); ++k) d[k] -= alpha[i] * hist[i].y[k];
    }
    const Pair& last = hist.back();
    const double gamma = vdot(last.s, last.y) / vdot(last.y, last.y);
    for (double& v : d) v *= gamma;
    for (std::size_t i = 0; i < hist.size(); ++i) {
      const double beta = hist[i].rho * vdot(hist[i].y, d);
      for (std::size_t k = 0; k < d.size(); ++k) d[k] += (alpha[i] - beta) * hist[i].s[k];
    }
  }
  for (double& v : d) v = -v;
  return d;
}

// Counts evaluations around any objective (minimize's Evaluator).
struct Eval {
  const gsb::LbfgsObjective& fn;
  int evaluations = 0;
  double operator()(const Vec& x, Vec& g) {
    ++evaluations;
    return fn(x, g);
  }
};

// A device failure inside the objective aborts the whole optimization.
struct DeviceFailure {
  gs_status status;
};

// The registration objective: one device evaluate() per call.
struct DeviceObjective {
  gs_ctx* ctx;
  const gs_config* cfg;
  int64_t n;
  const double* q0;
  const double* target;
  gs_report last{};
  gs_stats stats{};

  double operator()(const Vec& x, Vec& g) {
    g.assign(x.size(), 0.0);
    for (double v : x)
      if (!std::isfinite(v)) return kInf;  // MomentumSet rejects it (invalid_argument)
    gs_report r{};
    gs_stats s{};
    const gs_status st = gs_evaluate(ctx, cfg, n, q0, x.data(), target, &r, g.data(), &s);
    if (st == GS_NONFINITE || st == GS_INVALID_ARGUMENT) return kInf;
    if (st != GS_OK) throw DeviceFailure{st};
    last = r;
    stats.direct_interactions += s.direct_interactions;
    stats.approximated_interactions += s.approximated_interactions;
    stats.nodes_visited += s.nodes_visited;
    stats.traversal_queries += s.traversal_queries;
    stats.tree_build_ms += s.tree_build_ms;
    stats.forward_ms += s.forward_ms;
    stats.backward_ms += s.backward_ms;
    return r.total;
  }
};

// The same objective with device-resident inputs (evaluate_resident).
struct ResidentObjective {
  gs_ctx* ctx;
  const gs_config* cfg;
  int64_t n;
  gsb::DBuf q0, target;
  double box[6] = {0, 0, 0, 0, 0, 0};
  gs_report last{};
  gs_stats stats{};

  gs_status upload(const double* q0h, const double* th) {
    const size_t b = sizeof(double) * 3 * (size_t)n;
    if (q0.ensure(b) != GS_OK || target.ensure(b) != GS_OK) return GS_CUDA_ERROR;
    cudaStream_t st = gsb::context_stream(ctx);
    if (cudaMemcpyAsync(q0.ptr, q0h, b, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemcpyAsync(target.ptr, th, b, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return GS_CUDA_ERROR;
    gsb::host_box(q0h, n, box);
    return GS_OK;
  }

  double operator()(const double* x, double* g) {
    gs_report r{};
    gs_stats s{};
    const int st = gsb::evaluate_resident(ctx, cfg, n, q0.as<double>(), box, x, target.as<double>(),
                                          &r, g, &s);
    if (st == GS_NONFINITE || st == GS_INVALID_ARGUMENT) {  // rejected trial point: +inf, g = 0
      cudaMemsetAsync(g, 0, sizeof(double) * 3 * (size_t)n, gsb::context_stream(ctx));
      return kInf;
    }
    if (st != GS_OK) throw DeviceFailure{(gs_status)st};
    last = r;
    stats.direct_interactions += s.direct_interactions;
    stats.approximated_interactions += s.approximated_interactions;
    stats.nodes_visited += s.nodes_visited;
    stats.traversal_queries += s.traversal_queries;
    stats.tree_build_ms += s.tree_build_ms;
    stats.forward_ms += s.forward_ms;
    stats.backward_ms += s.backward_ms;
    return r.total;
  }
};

struct Step {
  bool ok = false;
  double f = kInf;
  Vec x, g;
};

Step wolfe(Eval& F, const Vec& x0, double f0, const Vec& g0, const Vec& d, double a0,
           const gs_opt_config& c) {
  Step out;
  const double slope0 = vdot(g0, d);
  if (slope0 >= 0.0) return out;
  auto point = [&](double a) {
    Vec x(x0.size());
    for (std::size_t i = 0; i < x.size(); ++i) x[i] = x0[i] + a * d[i];
    return x;
  };
  auto decreases = [&](double a, double fa) { return fa <= f0 + c.sufficient_decrease * a * slope0; };
  auto curvature_ok = [&](double slope) { return std::abs(slope) <= -c.curvature * slope0; };

  int trials = 0;
  double best_a = 0.0, best_f = f0;
  double a_prev = 0.0, f_prev = f0, a = a0;
  double lo = -1.0, hi = -1.0, f_lo = 0.0;
  bool bracketed = false;
  Vec g;
  while (trials < c.max_trials) {
    const double at = bracketed ? 0.5 * (lo + hi) : a;
    Vec x = point(at);
    const double fa = F(x, g);
    ++trials;
    const double slope = std::isfinite(fa) ? vdot(g, d) : 0.0;
    if (!bracketed) {
      if (!std::isfinite(fa) || !decreases(at, fa) || (trials > 1 && fa >= f_prev)) {
        lo = a_prev;
        f_lo = f_prev;
        hi = at;
        bracketed = true;
        continue;
      }
    } else if (!std::isfinite(fa) || !decreases(at, fa) || fa >= f_lo) {
      hi = at;
      continue;
    }
    if (fa < best_f) {
      best_a = at;
      best_f = fa;
    }
    if (curvature_ok(slope)) {
      out.ok = true;
      out.f = fa;
      out.x = std::move(x);
      out.g = std::move(g);
      return out;
    }
    if (!bracketed) {
      if (slope >= 0.0) {
        lo = at;
        f_lo = fa;
        hi = a_prev;
        bracketed = true;
        continue;
      }
      a_prev = at;
      f_prev = fa;
      a = 2.0 * at;
    } else {
      if (slope * (hi - lo) >= 0.0) hi = lo;
      lo = at;
      f_lo = fa;
    }
  }
  if (best_a > 0.0 && best_f < f0) {  // budget spent: re-evaluate the best decrease point
    Vec x = point(best_a);
    const double fb = F(x, g);
    if (std::isfinite(fb) && fb < f0) {
      out.ok = true;
      out.f = fb;
      out.x = std::move(x);
      out.g = std::move(g);
    }
  }
  return out;
}

}  // namespace

extern "C" {

gs_opt_config gs_default_opt_config(void) {
  gs_opt_config c;
  c.max_iterations = 200;
  c.memory = 10;
  c.gradient_tolerance = 1e-6;
  c.relative_objective_tolerance = 1e-9;
  c.sufficient_decrease = 1e-4;
  c.curvature = 0.9;
  c.max_trials = 20;
  return c;
}

}  // extern "C"

namespace gsb {

// minimize(), optimizer.cpp:215-299: L-BFGS from x0 with the strong-Wolfe
// search above; the same termination order and history rules.
LbfgsResult lbfgs_minimize(const LbfgsObjective& objective, std::vector<double> x0,
                           const gs_opt_config& oc, const LbfgsCallback& on_iterate) {
  const auto t0 = std::chrono::steady_clock::now();
  auto ms = [&] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  };
  Eval F{objective};
  LbfgsResult res;
  res.x = std::move(x0);
  Vec g;
  res.f = F(res.x, g);
  if (!std::isfinite(res.f)) throw NonFiniteStart{};
  res.grad_inf = vmax_abs(g);
  if (on_iterate) on_iterate(0, res.f, res.grad_inf, ms());
  std::deque<Pair> hist;
  res.reason = -1;
  for (int it = 1; it <= oc.max_iterations; ++it) {
    if (res.grad_inf <= oc.gradient_tolerance) {
      res.reason = GS_TERM_GRADIENT_TOLERANCE;
      break;
    }
    Vec d = direction(g, hist);
    if (vdot(g, d) >= 0.0) {  // stale curvature: restart from steepest descent
      hist.clear();
      d = g;
      for (double& v : d) v = -v;
    }
    const double a0 = hist.empty() ? 1.0 / std::max(1.0, res.grad_inf) : 1.0;
    Step s = wolfe(F, res.x, res.f, g, d, a0, oc);
    if (!s.ok) {
      res.reason = GS_TERM_LINE_SEARCH_FAILURE;
      break;
    }
    if (!std::isfinite(vmax_abs(s.g))) {
      res.reason = GS_TERM_NON_FINITE;
      break;
    }
    Pair pr;
    pr.s.resize(res.x.size());
    pr.y.resize(res.x.size());
    for (std::size_t k = 0; k < res.x.size(); ++k) {
      pr.s[k] = s.x[k] - res.x[k];
      pr.y[k] = s.g[k] - g[k];
    }
    const double sy = vdot(pr.s, pr.y);
    if (sy > 1e-10 * std::sqrt(vdot(pr.s, pr.s)) * std::sqrt(vdot(pr.y, pr.y))) {
      pr.rho = 1.0 / sy;
      hist.push_back(std::move(pr));
      if ((int)hist.size() > oc.memory) hist.pop_front();
    }
    const double f_prev = res.f;
    res.x = std::move(s.x);
    res.f = s.f;
    g = std::move(s.g);
    res.grad_inf = vmax_abs(g);
    res.iterations = it;
    if (on_iterate) on_iterate(it, res.f, res.grad_inf, ms());
    if (std::abs(f_prev - res.f) <= oc.relative_objective_tolerance * std::max(1.0, std::abs(res.f))) {
      res.reason = GS_TERM_OBJECTIVE_TOLERANCE;
      break;
    }
  }
  if (res.reason < 0)
    res.reason = res.grad_inf <= oc.gradient_tolerance ? GS_TERM_GRADIENT_TOLERANCE
                                                       : GS_TERM_MAX_ITERATIONS;
  res.evaluations = F.evaluations;
  return res;
}

}  // namespace gsb

extern "C" {

gs_status gs_optimize(gs_ctx* ctx, const gs_config* cfg, const gs_opt_config* oc, int64_t n,
                      const double* q0, const double* target, double* p_out, int32_t* reason,
                      int32_t* iterations, int32_t* evaluations, double* trace,
                      int32_t* trace_len, gs_stats* stats) {
  if (!ctx || !cfg || !oc || !q0 || !target || !p_out) return GS_INVALID_ARGUMENT;
  gs_status st = gs_validate_config(cfg, nullptr);
  if (st != GS_OK) return st;
  DeviceObjective F{ctx, cfg, n, q0, target};
  int32_t tl = 0;
  // trace row per iterate: iter,total,energy,attachment,grad_inf,wall_ms (optimizer.cpp:204-213)
  auto record = [&](int it, double, double ginf, double wall_ms) {
    if (!trace) return;
    double* r = trace + 6 * (size_t)tl;
    r[0] = it;
    r[1] = F.last.total;
    r[2] = F.last.energy;
    r[3] = F.last.attachment;
    r[4] = ginf;
    r[5] = wall_ms;
    ++tl;
  };
  gsb::LbfgsResult res;
  try {
    if (!gsb::context_is_multi(ctx)) {
      // device-resident state: q0 and the target uploaded once, every vector
      // of the search in HBM, evaluate() straight from them
      ResidentObjective R{ctx, cfg, n};
      const gs_status us = R.upload(q0, target);
      if (us != GS_OK) return us;
      auto rec = [&](int it, double f, double ginf, double wall_ms) {
        F.last = R.last;
        record(it, f, ginf, wall_ms);
      };
      const int s = gsb::lbfgs_minimize_device([&](const double* x, double* g) { return R(x, g); },
                                               3 * n, *oc, gsb::context_stream(ctx), rec, p_out,
                                               res);
      if (s != GS_OK) return (gs_status)s;
      F.stats = R.stats;
    } else {  // a multi-device context: host vectors, sharded evaluate()
      res = gsb::lbfgs_minimize([&](const Vec& x, Vec& g) { return F(x, g); },
                                Vec((size_t)3 * n, 0.0), *oc, record);
      std::copy(res.x.begin(), res.x.end(), p_out);
    }
  } catch (const DeviceFailure& e) {
    return e.status;
  } catch (const gsb::NonFiniteStart&) {
    return GS_NONFINITE;  // NonFiniteObjectiveAtStart
  } catch (const std::bad_alloc&) {
    return GS_INTERNAL;
  }
  if (reason) *reason = res.reason;
  if (iterations) *iterations = res.iterations;
  if (evaluations) *evaluations = res.evaluations;
  if (trace_len) *trace_len = tl;
  if (stats) *stats = F.stats;
  return GS_OK;
}

// Batched subjects (BASELINE config 5): B independent registrations, each on
// its own context (CUDA stream) and host thread so the device overlaps the
// subjects' kernels; no communication between subjects.
gs_status gs_optimize_batch(int device, const gs_config* cfg, const gs_opt_config* opt,
                            int32_t batch, const int64_t* n, const double* const* q0,
                            const double* const* target, double* const* p_out, int32_t* reasons,
                            int32_t* iterations, int32_t* evaluations, double* final_total) {
  if (!cfg || !opt || batch < 0 || !n || !q0 || !target || !p_out) return GS_INVALID_ARGUMENT;
  std::vector<gs_status> st((size_t)batch, GS_OK);
  std::vector<std::thread> pool;
  for (int32_t b = 0; b < batch; ++b)
    pool.emplace_back([&, b] {
      gs_status cs = GS_OK;
      cudaSetDevice(device);  // pooled contexts move between host threads
      gsb::set_bh_concurrency(batch);
      gs_ctx* c = ctx_pool().acquire(device, &cs);
      if (!c) {
        st[b] = cs;
        return;
      }
      std::vector<double> trace(6 * (size_t)(opt->max_iterations + 1));
      int32_t r = 0, it = 0, ev = 0, tl = 0;
      st[b] = gs_optimize(c, cfg, opt, n[b], q0[b], target[b], p_out[b], &r, &it, &ev,
                          trace.data(), &tl, nullptr);
      if (reasons) reasons[b] = r;
      if (iterations) iterations[b] = it;
      if (evaluations) evaluations[b] = ev;
      if (final_total) final_total[b] = tl > 0 ? trace[6 * (size_t)(tl - 1) + 1] : 0.0;
      ctx_pool().release(device, c);
    });
  for (auto& t : pool) t.join();
  for (gs_status s : st)
    if (s != GS_OK) return s;
  return GS_OK;
}

gs_status gs_evaluate_batch(int device, const gs_config* cfg, int32_t batch, const int64_t* n,
                            const double* const* q0, const double* const* p0,
                            const double* const* target, gs_report* reports,
                            double* const* grad_out, gs_stats* stats) {
  if (!cfg || batch < 0 || !n || !q0 || !p0 || !target || !reports || !grad_out)
    return GS_INVALID_ARGUMENT;
  std::vector<gs_status> st((size_t)batch, GS_OK);
  std::vector<std::thread> pool;
  for (int32_t b = 0; b < batch; ++b)
    pool.emplace_back([&, b] {
      gs_status cs = GS_OK;
      cudaSetDevice(device);  // pooled contexts move between host threads
      gsb::set_bh_concurrency(batch);
      gs_ctx* c = ctx_pool().acquire(device, &cs);
      if (!c) {
        st[b] = cs;
        return;
      }
      st[b] = gs_evaluate(c, cfg, n[b], q0[b], p0[b], target[b], reports + b, grad_out[b],
                          stats ? stats + b : nullptr);
      ctx_pool().release(device, c);
    });
  for (auto& t : pool) t.join();
  for (gs_status s : st)
    if (s != GS_OK) return s;
  return GS_OK;
}

}  // extern "C"
