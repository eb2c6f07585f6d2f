// C++ API parity checks: the reference's own test scenarios (proj/tests/
// test_kernel_exact.cpp, test_octree.cpp, test_bh_kernel.cpp,
// test_shooting.cpp), restated against paper_1907_04834_b200's geoshoot::
// headers -- i.e. what a reference user's code sees after switching to the
// B200 library. Run by tests/test_cpp_api.py on a GPU box; prints one line
// per check and exits non-zero on any failure.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "geoshoot/bh_kernel.hpp"
#include "geoshoot/optimizer.hpp"
#include "geoshoot/pipeline.hpp"
#include "geoshoot/shooting.hpp"

using namespace geoshoot;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    if (cond) ++g_pass;                                                  \
    else { ++g_fail; std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond); } \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static double u01(std::mt19937_64& r) { return static_cast<double>(r() >> 11) * 0x1.0p-53; }
static std::vector<Vec3> vecs(std::size_t n, double lo, double hi, std::uint64_t seed) {
  std::mt19937_64 r(seed);
  std::vector<Vec3> v;
  for (std::size_t i = 0; i < n; ++i)
    v.push_back({lo + (hi - lo) * u01(r), lo + (hi - lo) * u01(r), lo + (hi - lo) * u01(r)});
  return v;
}

static void kernel_exact() {
  CHECK(gaussian(0.0, 2.0) == 1.0);
  CHECK(std::abs(gaussian(6.0, 2.0) - std::exp(-4.5)) < 1e-17);
  const PointSet q1({{1.0, 2.0, 3.0}});
  const MomentumSet p1({{0.5, -1.0, 0.25}});
  const HamiltonianGradients g1 = hamiltonian_gradients(q1, p1, 3.0);
  CHECK(g1.dH_dp[0] == (Vec3{1.0, -2.0, 0.5}));
  CHECK(g1.dH_dq[0] == Vec3{});
  CHECK(std::abs(hamiltonian(PointSet({{0.3, -0.2, 1.0}}), MomentumSet({{1.0, 0, 0}}), 7.0) - 1.0) < 1e-15);
  CHECK(throws<DimensionMismatch>([] { hamiltonian(PointSet(vecs(3, 0, 1, 1)), MomentumSet::zeros(4), 1.0); }));
  // dH/dp = flow factor x velocity
  const PointSet q(vecs(8, 0, 3, 81));
  const MomentumSet p(vecs(8, -1, 1, 82));
  const HamiltonianGradients g = hamiltonian_gradients(q, p, 1.4);
  const std::vector<Vec3> v = exact_velocity(q, q, p, 1.4);
  for (std::size_t i = 0; i < 8; ++i) CHECK(norm(g.dH_dp[i] - flow_velocity_factor * v[i]) < 1e-12 * (1 + norm(g.dH_dp[i])));
  // finite differences of H (test_kernel_exact.cpp:143-164)
  const double h = 1e-5, sigma = 1.3;
  const PointSet qq(vecs(5, 0, 2, 51));
  const MomentumSet pp(vecs(5, -1, 1, 52));
  const HamiltonianGradients gg = hamiltonian_gradients(qq, pp, sigma);
  for (std::size_t i = 0; i < 5; ++i) {
    std::vector<Vec3> a = qq.data(), b = qq.data();
    a[i].x += h;
    b[i].x -= h;
    const double fd = (hamiltonian(PointSet(a), pp, sigma) - hamiltonian(PointSet(b), pp, sigma)) / (2 * h);
    CHECK(std::abs(gg.dH_dq[i].x - fd) <= 1e-6 * std::max({std::abs(fd), std::abs(gg.dH_dq[i].x), 1e-8}));
  }
}

static void octree() {
  std::vector<Vec3> corners;
  for (int i = 0; i < 8; ++i) corners.push_back({i & 1 ? 1.0 : -1.0, i & 2 ? 1.0 : -1.0, i & 4 ? 1.0 : -1.0});
  const Octree t = Octree::build(PointSet(corners), MomentumSet::zeros(8));
  CHECK(t.node_count() == 9 && t.root().count == 8 && !t.root().leaf);
  for (int c = 0; c < 8; ++c) {
    CHECK(t.root().children[c] != Octree::no_child);
    if (t.root().children[c] != Octree::no_child) {
      const auto& ch = t.node(static_cast<std::size_t>(t.root().children[c]));
      CHECK(ch.leaf && ch.count == 1 && corners[static_cast<std::size_t>(ch.first_point)] == corners[c]);
    }
  }
  // explicit root cell + insert (test_octree.cpp:112-144)
  Octree e({0, 0, 0}, {8, 8, 8});
  e.insert(0, {1, 1, 1}, {0.5, 0, 0});
  CHECK(e.root().leaf && e.root().count == 1);
  e.insert(1, {7, 7, 7}, {0, 0.5, 0});
  CHECK(!e.root().leaf && e.root().count == 2 && e.root().momentum_sum == (Vec3{0.5, 0.5, 0}));
  CHECK(throws<OutOfBounds>([&] { e.insert(2, {9, 0, 0}, {}); }));
  // bucket at the depth cap (test_octree.cpp:270-296)
  std::vector<Vec3> dup(10, Vec3{0.5, 0.5, 0.5});
  dup.push_back({2.0, 2.0, 2.0});
  const Octree b = Octree::build(PointSet(dup), MomentumSet(vecs(11, -1, 1, 66)));
  std::size_t max_chain = 0;
  for (std::size_t k = 0; k < b.node_count(); ++k) {
    if (!b.node(k).leaf) continue;
    std::size_t len = 0;
    for (std::int32_t i = b.node(k).first_point; i >= 0; i = b.next_point()[static_cast<std::size_t>(i)]) ++len;
    CHECK(len == b.node(k).count);
    max_chain = std::max(max_chain, len);
  }
  CHECK(max_chain == 10 && b.node_count() <= 2 * (Octree::max_depth + 2));
  // adjoint sums (test_octree.cpp:156-198)
  const std::size_t n = 50;
  Octree a = Octree::build(PointSet(vecs(n, 0, 5, 17)), MomentumSet(vecs(n, -1, 1, 18)));
  a.accumulate_adjoints(vecs(n, -2, 2, 19), vecs(n, -2, 2, 20));
  const std::vector<Vec3> al = vecs(n, -2, 2, 19);
  Vec3 s{};
  for (const Vec3& x : al) s += x;
  CHECK(norm(a.root().alpha_sum - s) <= 1e-12 * (1 + norm(s)));
  CHECK(throws<DimensionMismatch>([&] { a.accumulate_adjoints(std::vector<Vec3>(n - 1), std::vector<Vec3>(n)); }));
}

static void bh() {
  const double inf = std::numeric_limits<double>::infinity();
  const std::size_t n = 120;
  const double sigma = 1.1;
  const PointSet q(vecs(n, 0, 8, 301));
  const MomentumSet p(vecs(n, -1, 1, 302));
  const Octree tree = Octree::build(q, p);
  TraversalStats st;
  const HamiltonianGradients want = hamiltonian_gradients(q, p, sigma);
  const HamiltonianGradients got = bh_hamiltonian_gradients(tree, q, p, sigma, inf, &st);
  CHECK(st.approximated_interactions == 0 && st.direct_interactions == n * n);
  for (std::size_t i = 0; i < n; ++i) CHECK(norm(got.dH_dp[i] - want.dH_dp[i]) <= 1e-12 * (1 + norm(want.dH_dp[i])));
  const BhVelocity one = bh_velocity(Octree::build(PointSet({{1, 2, 3}}), MomentumSet({{0.5, -0.5, 1}})), {1, 2, 3}, 2.0, 1e-9);
  CHECK(one.velocity == (Vec3{0.5, -0.5, 1}) && one.stats.direct_interactions == 1);
  CHECK(throws<EmptyTree>([] { bh_velocity(Octree({0, 0, 0}, {1, 1, 1}), {0, 0, 0}, 1.0, 3.0); }));
  // envelope at 3 sigma (test_bh_kernel.cpp:185-205)
  const PointSet qe(vecs(150, 0, 15, 61));
  const MomentumSet pe(vecs(150, -1.5, 1.5, 161));
  const Octree te = Octree::build(qe, pe);
  const std::vector<Vec3> ve = exact_velocity(qe, qe, pe, 0.6);
  double mass = 0;
  for (const Vec3& v : pe) mass += norm(v);
  for (std::size_t i = 0; i < 150; i += 7) CHECK(norm(bh_velocity(te, qe[i], 0.6, 1.8).velocity - ve[i]) < std::exp(-4.5) * mass);
}

static ShootingConfig cfg(double sigma, double lambda, int T, Backend b = Backend::Exact) {
  ShootingConfig c;
  c.sigma = sigma;
  c.lambda = lambda;
  c.timesteps = T;
  c.backend = b;
  return c;
}

static void shooting() {
  const PointSet q(vecs(4, 0, 2, 401));
  const MomentumSet p(vecs(4, -0.3, 0.3, 402));
  for (int T : {1, 5, 40}) CHECK(shoot_forward(q, p, cfg(1, 1, T)).states.size() == static_cast<std::size_t>(T) + 1);
  const PointSet f({{0.5, -0.25, 2.0}});
  const MomentumSet fp({{1.0, 0, 0}});
  CHECK(norm(shoot_forward(f, fp, cfg(3, 1, 7)).final_state().q[0] - (f[0] + 2.0 * fp[0])) < 1e-12);
  // adjoint vs finite differences (test_shooting.cpp:174-200)
  const ShootingConfig c = cfg(1.1, 0.8, 10);
  const PointSet q3(vecs(3, 0, 2, 441)), t3(vecs(3, 0, 2, 443));
  const MomentumSet p3(vecs(3, -0.3, 0.3, 442));
  const std::vector<Vec3> grad = backward_gradient(shoot_forward(q3, p3, c), t3, c);
  const double h = 1e-5;
  for (std::size_t i = 0; i < 3; ++i) {
    std::vector<Vec3> hi = p3.data(), lo = p3.data();
    hi[i].y += h;
    lo[i].y -= h;
    const double fd = (objective(q3, MomentumSet(hi), t3, c).total - objective(q3, MomentumSet(lo), t3, c).total) / (2 * h);
    CHECK(std::abs(grad[i].y - fd) <= 1e-5 * std::max({std::abs(fd), std::abs(grad[i].y), 1e-6}));
  }
  // BH with infinite threshold == exact (test_shooting.cpp:236-253)
  const PointSet q6(vecs(60, 0, 5, 461)), t6(vecs(60, 0, 5, 463));
  const MomentumSet p6(vecs(60, -0.3, 0.3, 462));
  ShootingConfig bhc = cfg(1.2, 1, 8, Backend::BarnesHut);
  bhc.threshold_multiplier = std::numeric_limits<double>::infinity();
  const Evaluation a = evaluate(q6, p6, t6, cfg(1.2, 1, 8)), b = evaluate(q6, p6, t6, bhc);
  CHECK(std::abs(b.report.total - a.report.total) <= 1e-10 * std::abs(a.report.total));
  for (std::size_t i = 0; i < 60; ++i) CHECK(norm(b.gradient[i] - a.gradient[i]) <= 1e-10 * (1 + norm(a.gradient[i])));
  // determinism, non-finite, config errors, mismatch
  const Evaluation a2 = evaluate(q6, p6, t6, cfg(1.2, 1, 8));
  CHECK(a2.report.total == a.report.total);
  CHECK(throws<NonFiniteState>([] {
    shoot_forward(PointSet({{0, 0, 0}, {0.1, 0, 0}}), MomentumSet({{1e200, 0, 0}, {1e200, 0, 0}}), cfg(0.05, 1, 4));
  }));
  bool all4 = false;
  try {
    ShootingConfig bad = cfg(-1, 0, 0);
    bad.threshold_multiplier = 0;
    validate_config(bad);
  } catch (const ConfigError& e) {
    all4 = e.violations.size() == 4;
  }
  CHECK(all4);
  const GeodesicTrajectory tr = shoot_forward(q6, p6, cfg(1.2, 1, 8));
  CHECK(throws<ConfigMismatch>([&] { warp_points(tr, q6, cfg(1.2, 1, 9)); }));
  const PointSet w = warp_points(tr, q6, cfg(1.2, 1, 8));
  for (std::size_t i = 0; i < 60; ++i) CHECK(norm(w[i] - tr.final_state().q[i]) < 1e-10);
}

static void adjacent() {
  // optimize (optimizer.cpp:301-351): objective decreases from p0 = 0
  const PointSet q(vecs(40, 0, 6, 501));
  std::vector<Vec3> moved = q.data();
  for (Vec3& v : moved) v += Vec3{0.3, -0.2, 0.1};
  ShootingConfig c = cfg(2.0, 1.0, 6);
  c.optimizer.max_iterations = 10;
  auto [p, trace] = optimize(q, PointSet(moved), c);
  CHECK(trace.records.size() >= 2 && trace.records.back().total < trace.records.front().total);
  CHECK(p.size() == q.size());
  // files: %.17g round trip (pipeline_io.cpp:117-149)
  const std::string f = "/tmp/geoshoot_b200_test_api.vtk";
  write_points(q, f, format_for_path(f), {"title"});
  const PointSet back = read_points(f, PointFormat::LegacyPolydataAscii);
  bool same = back.size() == q.size();
  for (std::size_t i = 0; same && i < q.size(); ++i) same = back[i] == q[i];
  CHECK(same);
  // procrustes: exact recovery of a translation
  const ProcrustesResult pr = procrustes_align(q, PointSet(moved));
  CHECK(norm(pr.transform.translation - Vec3{0.3, -0.2, 0.1}) < 1e-12);
  CHECK(throws<DegenerateConfiguration>([] {
    procrustes_align(PointSet({{0, 0, 0}, {1, 1, 1}}), PointSet({{0, 0, 0}, {1, 1, 1}}));
  }));
}

int main() {
  kernel_exact();
  octree();
  bh();
  shooting();
  adjacent();
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
