// api.cpp -- the reference's C++ API (include/geoshoot/*.hpp) as a thin shim
// over the C ABI: arguments are validated like the reference does, arrays
// are passed as the reinterpret_cast'ed Vec3 buffers, gs_status codes are
// mapped back to the reference's exception types. No arithmetic of the hot
// path happens here.
#include <algorithm>
#include <cstdio>
#include <ostream>
#include <cstdlib>
#include <cstring>
#include <string>

#include "geoshoot/bh_kernel.hpp"
#include "geoshoot/core.hpp"
#include "geoshoot/kernel_exact.hpp"
#include "geoshoot/octree.hpp"
#include "geoshoot/optimizer.hpp"
#include "geoshoot/pipeline.hpp"
#include "geoshoot/shooting.hpp"
#include "geoshoot_b200.h"
#include "lbfgs.h"

namespace geoshoot {
namespace {

const double* raw(const std::vector<Vec3>& v) { return reinterpret_cast<const double*>(v.data()); }
double* raw(std::vector<Vec3>& v) { return reinterpret_cast<double*>(v.data()); }

// one device context per host thread: device GEOSHOOT_DEVICE (default 0), or
// -- GEOSHOOT_DEVICES="0,1,2,3" -- a multi-device context whose shooting calls
// (shoot_forward, objective, evaluate, optimize) shard the targets across them
struct Ctx {
  gs_ctx* c = nullptr;
  ~Ctx() {
    if (c) gs_destroy(c);
  }
};

gs_ctx* ctx() {
  thread_local Ctx holder;
  if (!holder.c) {
    gs_status st = GS_OK;
    if (const char* list = std::getenv("GEOSHOOT_DEVICES")) {
      std::vector<int32_t> devs;
      for (const char* p = list; *p;) {
        char* end = nullptr;
        const long v = std::strtol(p, &end, 10);
        if (end == p) break;
        devs.push_back((int32_t)v);
        p = *end == ',' ? end + 1 : end;
      }
      holder.c = gs_create_multi((int32_t)devs.size(), devs.data(), &st);
    } else {
      const char* env = std::getenv("GEOSHOOT_DEVICE");
      holder.c = gs_create(env ? std::atoi(env) : 0, &st);
    }
    if (!holder.c) throw DeviceError(std::string("geoshoot: no B200 device: ") + gs_last_error(nullptr));
  }
  return holder.c;
}

thread_local Precision g_precision = Precision::F64;

void check(gs_status st) {
  if (st == GS_OK) return;
  const std::string msg = gs_last_error(nullptr);
  switch (st) {
    case GS_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
    case GS_CONFIG_ERROR: {
      std::vector<ConfigViolation> v;
      const uint32_t m = gs_last_config_violations(nullptr);
      for (int k = 0; k < 4; ++k)
        if (m & (1u << k)) v.push_back(static_cast<ConfigViolation>(k));
      throw ConfigError(std::move(v));
    }
    case GS_NONFINITE: throw NonFiniteState(gs_last_nonfinite_step(nullptr));
    case GS_CONFIG_MISMATCH: throw ConfigMismatch(msg);
    case GS_EMPTY_TREE: throw EmptyTree(msg);
    case GS_OUT_OF_BOUNDS: throw OutOfBounds(msg);
    case GS_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case GS_DEGENERATE: throw DegenerateConfiguration(msg);
    default: throw DeviceError("geoshoot device error " + std::to_string(st) + ": " + msg);
  }
}

int32_t prec_of(Precision p) { return p == Precision::F32 ? GS_F32 : GS_F64; }

gs_config to_c(const ShootingConfig& c) {
  gs_config g;
  g.sigma = c.sigma;
  g.lambda = c.lambda;
  g.timesteps = c.timesteps;
  g.backend = c.backend == Backend::BarnesHut ? GS_BARNES_HUT : GS_EXACT;
  g.threshold_multiplier = c.threshold_multiplier;
  g.integrator = c.integrator == Integrator::RK4 ? GS_RK4 : GS_EULER;
  g.precision = prec_of(c.precision);
  g.literal_mean_dot = c.literal_mean_dot ? 1 : 0;
  g.flags = c.exact_underflow_cutoff ? GS_FLAG_EXACT_CUTOFF : 0u;
  return g;
}

TraversalStats to_traversal(const gs_stats& s) {
  TraversalStats t;
  t.direct_interactions = s.direct_interactions;
  t.approximated_interactions = s.approximated_interactions;
  t.nodes_visited = s.nodes_visited;
  return t;
}

std::vector<Vec3> flat_states(const GeodesicTrajectory& tr, bool momenta) {
  std::vector<Vec3> out;
  out.reserve(tr.states.size() * tr.point_count());
  for (const auto& s : tr.states) {
    const auto& v = momenta ? s.p.data() : s.q.data();
    out.insert(out.end(), v.begin(), v.end());
  }
  return out;
}

}  // namespace

int default_thread_count() { return 1; }

ValidatedConfig validate_config(const ShootingConfig& config) {
  const gs_config g = to_c(config);
  uint32_t mask = 0;
  check(gs_validate_config(&g, &mask));
  return ValidatedConfig{config};
}

void set_kernel_precision(Precision p) { g_precision = p; }
Precision kernel_precision() { return g_precision; }

// ---- kernel_exact -------------------------------------------------------------
double hamiltonian(const PointSet& q, const MomentumSet& p, double sigma) {
  require_aligned(q.size(), p.size(), "hamiltonian");
  double h = 0.0;
  check(gs_hamiltonian(ctx(), prec_of(g_precision), (int64_t)q.size(), raw(q.data()), raw(p.data()),
                       sigma, &h));
  return h;
}

double hamiltonian_with_gradients(const PointSet& q, const MomentumSet& p, double sigma,
                                  HamiltonianGradients& out) {
  require_aligned(q.size(), p.size(), "hamiltonian_gradients");
  out.dH_dp.assign(q.size(), Vec3{});
  out.dH_dq.assign(q.size(), Vec3{});
  double h = 0.0;
  check(gs_exact_rhs(ctx(), prec_of(g_precision), (int64_t)q.size(), raw(q.data()), raw(p.data()),
                     sigma, raw(out.dH_dp), raw(out.dH_dq), &h));
  return h;
}

HamiltonianGradients hamiltonian_gradients(const PointSet& q, const MomentumSet& p, double sigma) {
  HamiltonianGradients g;
  hamiltonian_with_gradients(q, p, sigma, g);
  return g;
}

std::vector<Vec3> exact_velocity(const PointSet& q_eval, const PointSet& q_src,
                                 const MomentumSet& p_src, double sigma) {
  require_aligned(q_src.size(), p_src.size(), "exact_velocity");
  std::vector<Vec3> v(q_eval.size());
  check(gs_exact_velocity(ctx(), prec_of(g_precision), (int64_t)q_eval.size(), raw(q_eval.data()),
                          (int64_t)q_src.size(), raw(q_src.data()), raw(p_src.data()), sigma,
                          raw(v)));
  return v;
}

HessianProducts hessian_products(const PointSet& q, const MomentumSet& p,
                                 const std::vector<Vec3>& alpha, const std::vector<Vec3>& beta,
                                 double sigma) {
  require_aligned(q.size(), p.size(), "hessian_products");
  require_aligned(q.size(), alpha.size(), "hessian_products(alpha)");
  require_aligned(q.size(), beta.size(), "hessian_products(beta)");
  HessianProducts h;
  for (auto* v : {&h.pq_alpha, &h.pp_alpha, &h.qq_beta, &h.qp_beta}) v->assign(q.size(), Vec3{});
  check(gs_hessian_products(ctx(), prec_of(g_precision), (int64_t)q.size(), raw(q.data()),
                            raw(p.data()), raw(alpha), raw(beta), sigma, raw(h.pq_alpha),
                            raw(h.pp_alpha), raw(h.qq_beta), raw(h.qp_beta)));
  return h;
}

// ---- octree ------------------------------------------------------------------
Octree::Octree(const Vec3& cell_min, const Vec3& cell_max)
    : root_min_(cell_min), root_max_(cell_max), explicit_root_(true) {
  Node r;
  r.cell_min = cell_min;
  r.cell_max = cell_max;
  nodes_.push_back(r);
}

Octree::~Octree() {
  if (dev_) gs_tree_free(dev_);
}

Octree::Octree(Octree&& o) noexcept { *this = std::move(o); }

Octree& Octree::operator=(Octree&& o) noexcept {
  if (this != &o) {
    if (dev_) gs_tree_free(dev_);
    nodes_ = std::move(o.nodes_);
    points_ = std::move(o.points_);
    momenta_ = std::move(o.momenta_);
    next_point_ = std::move(o.next_point_);
    root_min_ = o.root_min_;
    root_max_ = o.root_max_;
    explicit_root_ = o.explicit_root_;
    dirty_ = o.dirty_;
    dev_ = o.dev_;
    dev_alpha_ = o.dev_alpha_;
    dev_beta_ = o.dev_beta_;
    o.dev_ = nullptr;
    o.dirty_ = false;
  }
  return *this;
}

Octree Octree::build(const PointSet& q, const MomentumSet& p) {
  require_aligned(q.size(), p.size(), "Octree::build");
  Octree t;
  t.points_ = q.data();
  t.momenta_ = p.data();
  t.rebuild(false);
  return t;
}

void Octree::rebuild(bool explicit_root) const {
  dirty_ = false;
  dev_alpha_ = dev_beta_ = nullptr;
  if (dev_) {
    gs_tree_free(dev_);
    dev_ = nullptr;
  }
  if (points_.empty()) return;
  const int64_t n = (int64_t)points_.size();
  if (explicit_root) {
    const double lo[3] = {root_min_.x, root_min_.y, root_min_.z};
    const double hi[3] = {root_max_.x, root_max_.y, root_max_.z};
    check(gs_tree_build_in_cell(ctx(), prec_of(g_precision), n, raw(points_), raw(momenta_), lo, hi,
                                &dev_));
  } else {
    check(gs_tree_build(ctx(), prec_of(g_precision), n, raw(points_), raw(momenta_), &dev_));
  }
  mirror();
}

// Host mirror of the device nodes in the reference's Node layout.
void Octree::mirror() const {
  const int64_t n = (int64_t)points_.size();
  const int64_t m = gs_tree_node_count(dev_);
  std::vector<int32_t> order(n), level(m), parent(m), skip(m), range(2 * m);
  std::vector<uint64_t> kh(n), kl(n);
  std::vector<double> boxes(12 * m), sums(12 * m);
  std::vector<uint32_t> count(m);
  check(gs_tree_download(dev_, order.data(), kh.data(), kl.data(), level.data(), parent.data(),
                         skip.data(), range.data(), boxes.data(), sums.data(), count.data()));
  nodes_.assign(m, Node{});
  next_point_.assign(n, -1);
  auto v3 = [](const double* d) { return Vec3{d[0], d[1], d[2]}; };
  for (int64_t k = 0; k < m; ++k) {
    Node& nd = nodes_[k];
    nd.cell_min = v3(&boxes[12 * k]);
    nd.cell_max = v3(&boxes[12 * k + 3]);
    nd.actual_min = v3(&boxes[12 * k + 6]);
    nd.actual_max = v3(&boxes[12 * k + 9]);
    nd.position_sum = v3(&sums[12 * k]);
    nd.momentum_sum = v3(&sums[12 * k + 3]);
    nd.alpha_sum = v3(&sums[12 * k + 6]);
    nd.beta_sum = v3(&sums[12 * k + 9]);
    nd.count = count[k];
    nd.leaf = skip[k] == k + 1 && (count[k] == 1 || level[k] == max_depth);
    if (nd.leaf) {  // chain newest first (reference octree.cpp:93-97)
      std::vector<int32_t> members(order.begin() + range[2 * k], order.begin() + range[2 * k + 1] + 1);
      std::sort(members.begin(), members.end(), std::greater<int32_t>());
      nd.first_point = members.front();
      for (size_t j = 0; j + 1 < members.size(); ++j) next_point_[members[j]] = members[j + 1];
    }
  }
  for (int64_t k = 1; k < m; ++k) {  // child slot = octant of the child cell in its parent
    Node& par = nodes_[parent[k]];
    par.children[octant_of(par, 0.5 * (nodes_[k].cell_min + nodes_[k].cell_max))] = (int32_t)k;
  }
}

void Octree::insert(std::uint32_t index, const Vec3& position, const Vec3& momentum) {
  const Node& r = nodes_.front();
  if (!(position.x >= r.cell_min.x && position.x <= r.cell_max.x && position.y >= r.cell_min.y &&
        position.y <= r.cell_max.y && position.z >= r.cell_min.z && position.z <= r.cell_max.z))
    throw OutOfBounds("Octree::insert: point outside the root cell");
  if (index != points_.size())
    throw std::invalid_argument("Octree::insert: points must arrive in index order");
  points_.push_back(position);
  momenta_.push_back(momentum);
  if (!explicit_root_) {
    root_min_ = r.cell_min;
    root_max_ = r.cell_max;
    explicit_root_ = true;
  }
  dirty_ = true;  // built once, on the next use (sync)
}

void Octree::accumulate_adjoints(const std::vector<Vec3>& alpha, const std::vector<Vec3>& beta) {
  require_aligned(points_.size(), alpha.size(), "accumulate_adjoints(alpha)");
  require_aligned(points_.size(), beta.size(), "accumulate_adjoints(beta)");
  sync();
  check(gs_tree_accumulate_adjoints(dev_, raw(alpha), raw(beta)));
  dev_alpha_ = alpha.data();
  dev_beta_ = beta.data();
  mirror();
}

double Octree::min_distance(const Node& nd, const Vec3& x) {
  const double dx = std::max({nd.actual_min.x - x.x, 0.0, x.x - nd.actual_max.x});
  const double dy = std::max({nd.actual_min.y - x.y, 0.0, x.y - nd.actual_max.y});
  const double dz = std::max({nd.actual_min.z - x.z, 0.0, x.z - nd.actual_max.z});
  return std::sqrt(dx * dx + dy * dy + dz * dz);
}

int Octree::octant_of(const Node& nd, const Vec3& x) {
  const Vec3 c = 0.5 * (nd.cell_min + nd.cell_max);
  return (x.x >= c.x ? 1 : 0) | (x.y >= c.y ? 2 : 0) | (x.z >= c.z ? 4 : 0);
}

gs_tree* Octree::device() const {
  sync();
  return dev_;
}

// ---- bh_kernel ----------------------------------------------------------------
namespace {
void require_tree(const Octree& t) {
  if (t.point_count() == 0 || !t.device()) throw EmptyTree("Barnes-Hut query on an empty tree");
}
}  // namespace

void set_bh_literal_mean_dot(bool enable) { check(gs_set_literal_mean_dot(ctx(), enable ? 1 : 0)); }

BhVelocity bh_velocity(const Octree& tree, const Vec3& x, double sigma, double threshold) {
  require_tree(tree);
  BhVelocity out;
  gs_stats st{};
  check(gs_bh_velocity(tree.device(), 1, &x.x, sigma, threshold, &out.velocity.x, &st));
  out.stats = to_traversal(st);
  return out;
}

HamiltonianGradients bh_hamiltonian_gradients(const Octree& tree, const PointSet& q,
                                              const MomentumSet& p, double sigma, double threshold,
                                              TraversalStats* stats) {
  require_aligned(q.size(), p.size(), "bh_hamiltonian_gradients");
  require_aligned(q.size(), tree.point_count(), "bh_hamiltonian_gradients(tree)");
  require_tree(tree);
  HamiltonianGradients g;
  g.dH_dp.assign(q.size(), Vec3{});
  g.dH_dq.assign(q.size(), Vec3{});
  gs_stats st{};
  check(gs_bh_rhs(tree.device(), sigma, threshold, raw(g.dH_dp), raw(g.dH_dq), &st));
  if (stats) stats->merge(to_traversal(st));
  return g;
}

BhPointGradients bh_point_gradients(const Octree& tree, const Vec3& x, const Vec3& px, double sigma,
                                    double threshold, TraversalStats* stats) {
  // one query of the batched device traversal (gs_bh_point_gradients): any
  // (x, px), tree point or not
  require_tree(tree);
  BhPointGradients out;
  gs_stats st{};
  check(gs_bh_point_gradients(tree.device(), 1, &x.x, &px.x, sigma, threshold, &out.dH_dp.x,
                              &out.dH_dq.x, &st));
  if (stats) stats->merge(to_traversal(st));
  return out;
}

BhPointHessianProducts bh_point_hessian_products(const Octree& tree, const Vec3& qi,
                                                 const Vec3& pi, const Vec3& alpha_i,
                                                 const Vec3& beta_i,
                                                 const std::vector<Vec3>& alpha,
                                                 const std::vector<Vec3>& beta, double sigma,
                                                 double threshold, TraversalStats* stats) {
  require_tree(tree);
  require_aligned(tree.point_count(), alpha.size(), "bh_point_hessian_products(alpha)");
  require_aligned(tree.point_count(), beta.size(), "bh_point_hessian_products(beta)");
  // Direct terms read alpha/beta by source index. The device already holds the
  // arrays of the last annotation / upload; re-send them only when the caller
  // passes other arrays, so a per-point loop over i (run_backward's pattern,
  // shooting.cpp:177-190) costs O(traversal) per call, not O(N).
  const bool same = alpha.data() == tree.device_alpha() && beta.data() == tree.device_beta();
  BhPointHessianProducts out;
  gs_stats st{};
  check(gs_bh_point_hessian_products(tree.device(), 1, &qi.x, &pi.x, &alpha_i.x, &beta_i.x,
                                     same ? nullptr : raw(alpha), same ? nullptr : raw(beta),
                                     sigma, threshold, &out.pq_alpha.x, &out.pp_alpha.x,
                                     &out.qq_beta.x, &out.qp_beta.x, &st));
  tree.note_device_adjoints(alpha.data(), beta.data());
  if (stats) stats->merge(to_traversal(st));
  return out;
}

double bh_hamiltonian(const Octree& tree, const PointSet& q, const MomentumSet& p, double sigma,
                      double threshold, TraversalStats* stats) {
  require_tree(tree);
  require_aligned(q.size(), p.size(), "bh_hamiltonian");
  require_aligned(q.size(), tree.point_count(), "bh_hamiltonian(tree)");
  double h = 0.0;
  gs_stats st{};
  check(gs_bh_hamiltonian(tree.device(), sigma, threshold, &h, &st));
  if (stats) stats->merge(to_traversal(st));
  return h;
}

HessianProducts bh_hessian_products(const Octree& tree, const PointSet& q, const MomentumSet& p,
                                    const std::vector<Vec3>& alpha, const std::vector<Vec3>& beta,
                                    double sigma, double threshold, TraversalStats* stats) {
  require_aligned(q.size(), p.size(), "bh_hessian_products");
  require_aligned(q.size(), alpha.size(), "bh_hessian_products(alpha)");
  require_aligned(q.size(), beta.size(), "bh_hessian_products(beta)");
  require_aligned(q.size(), tree.point_count(), "bh_hessian_products(tree)");
  require_tree(tree);
  HessianProducts h;
  for (auto* v : {&h.pq_alpha, &h.pp_alpha, &h.qq_beta, &h.qp_beta}) v->assign(q.size(), Vec3{});
  gs_stats st{};
  check(gs_bh_hessian_products(tree.device(), raw(alpha), raw(beta), sigma, threshold,
                               raw(h.pq_alpha), raw(h.pp_alpha), raw(h.qq_beta), raw(h.qp_beta),
                               &st));
  tree.note_device_adjoints(alpha.data(), beta.data());
  if (stats) stats->merge(to_traversal(st));
  return h;
}

// ---- shooting -----------------------------------------------------------------
GeodesicTrajectory shoot_forward(const PointSet& q0, const MomentumSet& p0,
                                 const ShootingConfig& config) {
  validate_config(config);
  require_aligned(q0.size(), p0.size(), "shoot_forward");
  const gs_config c = to_c(config);
  const std::size_t n = q0.size(), T = (std::size_t)config.timesteps;
  std::vector<Vec3> tq(n * (T + 1)), tp(n * (T + 1));
  check(gs_shoot_forward(ctx(), &c, (int64_t)n, raw(q0.data()), raw(p0.data()), raw(tq), raw(tp),
                         nullptr, nullptr, nullptr, nullptr));
  GeodesicTrajectory tr;
  tr.states.reserve(T + 1);
  for (std::size_t k = 0; k <= T; ++k)
    tr.states.push_back({PointSet(std::vector<Vec3>(tq.begin() + k * n, tq.begin() + (k + 1) * n)),
                         MomentumSet(std::vector<Vec3>(tp.begin() + k * n, tp.begin() + (k + 1) * n))});
  return tr;
}

ObjectiveReport objective(const PointSet& q0, const MomentumSet& p0, const PointSet& target,
                          const ShootingConfig& config) {
  validate_config(config);
  require_aligned(q0.size(), p0.size(), "shoot_forward");
  require_aligned(q0.size(), target.size(), "objective(target)");
  const gs_config c = to_c(config);
  gs_report r{};
  check(gs_objective(ctx(), &c, (int64_t)q0.size(), raw(q0.data()), raw(p0.data()),
                     raw(target.data()), &r));
  return {r.energy, r.attachment, r.total, r.residual_sse};
}

std::vector<Vec3> backward_gradient(const GeodesicTrajectory& tr, const PointSet& target,
                                    const ShootingConfig& config) {
  validate_config(config);
  if (tr.states.size() != static_cast<std::size_t>(config.timesteps) + 1)
    throw ConfigMismatch("backward_gradient: trajectory length != timesteps + 1");
  require_aligned(tr.point_count(), target.size(), "backward_gradient(target)");
  const gs_config c = to_c(config);
  const std::vector<Vec3> tq = flat_states(tr, false), tp = flat_states(tr, true);
  std::vector<Vec3> g(target.size());
  check(gs_backward_gradient(ctx(), &c, (int64_t)tr.point_count(), (int32_t)tr.states.size(),
                             raw(tq), raw(tp), raw(target.data()), raw(g)));
  return g;
}

PointSet warp_points(const GeodesicTrajectory& tr, const PointSet& x, const ShootingConfig& config) {
  validate_config(config);
  if (tr.states.size() != static_cast<std::size_t>(config.timesteps) + 1)
    throw ConfigMismatch("warp_points: trajectory length != timesteps + 1");
  const gs_config c = to_c(config);
  const std::vector<Vec3> tq = flat_states(tr, false), tp = flat_states(tr, true);
  std::vector<Vec3> y(x.size());
  check(gs_warp_points(ctx(), &c, (int64_t)tr.point_count(), (int32_t)tr.states.size(), raw(tq),
                       raw(tp), (int64_t)x.size(), raw(x.data()), raw(y)));
  return PointSet(std::move(y));
}

Evaluation evaluate(const PointSet& q0, const MomentumSet& p0, const PointSet& target,
                    const ShootingConfig& config, int) {
  validate_config(config);
  require_aligned(q0.size(), p0.size(), "shoot_forward");
  require_aligned(q0.size(), target.size(), "objective(target)");
  const gs_config c = to_c(config);
  gs_report r{};
  gs_stats st{};
  Evaluation ev;
  ev.gradient.assign(q0.size(), Vec3{});
  check(gs_evaluate(ctx(), &c, (int64_t)q0.size(), raw(q0.data()), raw(p0.data()),
                    raw(target.data()), &r, raw(ev.gradient), &st));
  ev.report = {r.energy, r.attachment, r.total, r.residual_sse};
  ev.stats.tree_build_ms = st.tree_build_ms;
  ev.stats.forward_ms = st.forward_ms;
  ev.stats.backward_ms = st.backward_ms;
  ev.stats.traversal = to_traversal(st);
  ev.stats.traversal_queries = st.traversal_queries;
  return ev;
}

// ---- point-cloud files ----------------------------------------------------------
namespace {
void io_check(gs_status st) {
  if (st == GS_OK) return;
  const std::string msg = gs_last_io_error();
  if (st == GS_PARSE_ERROR) {
    const std::string prefix = "line " + std::to_string(gs_last_parse_line()) + ": ";
    throw ParseError((std::size_t)gs_last_parse_line(),
                     msg.rfind(prefix, 0) == 0 ? msg.substr(prefix.size()) : msg);
  }
  if (st == GS_UNSUPPORTED_FORMAT) throw UnsupportedFormat(msg);
  if (st == GS_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
int32_t fmt_of(PointFormat f) { return f == PointFormat::LegacyPolydataAscii ? GS_FORMAT_VTK : GS_FORMAT_XYZ; }
}  // namespace

PointFormat format_for_path(const std::string& path) {
  return gs_format_for_path(path.c_str()) == GS_FORMAT_VTK ? PointFormat::LegacyPolydataAscii
                                                            : PointFormat::XyzText;
}

PointSet read_points(const std::string& path, PointFormat format) {
  int64_t n = 0;
  io_check(gs_read_points(path.c_str(), fmt_of(format), nullptr, 0, &n));
  std::vector<Vec3> v((std::size_t)n);
  io_check(gs_read_points(path.c_str(), fmt_of(format), raw(v), n, &n));
  return PointSet(std::move(v));
}

void write_points(const PointSet& points, const std::string& path, PointFormat format,
                  const std::vector<std::string>& header_comments) {
  std::vector<const char*> h;
  for (const auto& s : header_comments) h.push_back(s.c_str());
  io_check(gs_write_points(path.c_str(), fmt_of(format), (int64_t)points.size(), raw(points.data()),
                           h.data(), (int32_t)h.size()));
}

// ---- rigid pre-alignment ---------------------------------------------------------
ProcrustesResult procrustes_align(const PointSet& source, const PointSet& target) {
  require_aligned(source.size(), target.size(), "procrustes_align");
  double R[9], t[3];
  std::vector<Vec3> y(source.size());
  check(gs_procrustes_align(ctx(), (int64_t)source.size(), raw(source.data()), raw(target.data()),
                            R, t, raw(y)));
  RigidTransform tf;
  for (int r = 0; r < 3; ++r) tf.rotation_rows[r] = {R[3 * r], R[3 * r + 1], R[3 * r + 2]};
  tf.translation = {t[0], t[1], t[2]};
  return {tf, PointSet(std::move(y))};
}

// ---- optimizer ------------------------------------------------------------------
const char* to_string(TerminationReason r) {
  static const char* names[] = {"gradient_tolerance", "objective_tolerance", "max_iterations",
                                "line_search_failure", "non_finite"};
  return names[static_cast<int>(r)];
}

void OptimizationTrace::write_csv(std::ostream& os) const {
  os << "iter,total,energy,attachment,grad_inf,wall_ms\n";
  char line[256];
  for (const TraceRecord& r : records) {
    std::snprintf(line, sizeof line, "%d,%.17g,%.17g,%.17g,%.17g,%.3f\n", r.iteration, r.total,
                  r.energy, r.attachment, r.grad_inf, r.wall_ms);
    os << line;
  }
}

namespace {
gs_opt_config to_c(const OptimizerConfig& o) {
  gs_opt_config oc = gs_default_opt_config();
  oc.max_iterations = o.max_iterations;
  oc.memory = o.memory;
  oc.gradient_tolerance = o.gradient_tolerance;
  oc.relative_objective_tolerance = o.relative_objective_tolerance;
  oc.sufficient_decrease = o.line_search.sufficient_decrease;
  oc.curvature = o.line_search.curvature;
  oc.max_trials = o.line_search.max_trials;
  return oc;
}
}  // namespace

MinimizeResult minimize(const ObjectiveFn& objective, std::vector<double> x0,
                        const OptimizerConfig& config, const IterateCallback& on_iterate) {
  gsb::LbfgsResult r;
  try {
    r = gsb::lbfgs_minimize(objective, std::move(x0), to_c(config), on_iterate);
  } catch (const gsb::NonFiniteStart&) {
    throw NonFiniteObjectiveAtStart("objective is non-finite at the start point");
  }
  MinimizeResult out;
  out.x = std::move(r.x);
  out.f = r.f;
  out.grad_inf = r.grad_inf;
  out.reason = static_cast<TerminationReason>(r.reason);
  out.iterations = r.iterations;
  out.evaluations = r.evaluations;
  return out;
}

std::pair<MomentumSet, OptimizationTrace> optimize(const PointSet& q0, const PointSet& target,
                                                   const ShootingConfig& config,
                                                   EvalStats* eval_stats, int) {
  validate_config(config);
  require_aligned(q0.size(), target.size(), "optimize");
  const gs_config c = to_c(config);
  const gs_opt_config oc = to_c(config.optimizer);
  const std::size_t n = q0.size();
  std::vector<Vec3> p(n);
  std::vector<double> trace(6 * (std::size_t)(oc.max_iterations + 1));
  int32_t reason = 0, iters = 0, evals = 0, tl = 0;
  gs_stats st{};
  const gs_status s = gs_optimize(ctx(), &c, &oc, (int64_t)n, raw(q0.data()), raw(target.data()),
                                  raw(p), &reason, &iters, &evals, trace.data(), &tl, &st);
  if (s == GS_NONFINITE) throw NonFiniteObjectiveAtStart("objective is non-finite at the start point");
  check(s);
  OptimizationTrace tr;
  tr.reason = static_cast<TerminationReason>(reason);
  for (int32_t k = 0; k < tl; ++k) {
    const double* r = &trace[6 * (std::size_t)k];
    tr.records.push_back({(int)r[0], r[1], r[2], r[3], r[4], r[5]});
  }
  if (eval_stats) {
    EvalStats es;
    es.tree_build_ms = st.tree_build_ms;
    es.forward_ms = st.forward_ms;
    es.backward_ms = st.backward_ms;
    es.traversal = to_traversal(st);
    es.traversal_queries = st.traversal_queries;
    eval_stats->merge(es);
  }
  return {MomentumSet(std::move(p)), std::move(tr)};
}

}  // namespace geoshoot
