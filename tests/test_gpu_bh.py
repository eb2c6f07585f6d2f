"""Parity of the octree build and Barnes-Hut traversal against the reference.

* Morton keys and the leaf order are integer work: bit-exact against the
  oracle's midpoint replay (oracle/port.c) and the reference octree's own
  depth-first leaf order (oracle/_ref).
* Topology, counts and tight boxes: bit-exact as multisets against the
  reference node set; position/momentum sums to 1e-12 relative (summation
  order differs, test_octree.cpp:263-266).
* Traversal: per-query (direct, approximated, visited) counts EXACTLY equal to
  the reference's; FP64 values to 1e-12, FP32 (FP32-rounded inputs) to 1e-5.
"""
import os

import numpy as np
import pytest

from paper_1907_04834_b200 import BARNES_HUT, EXACT, F32, F64, RK4, ShootingConfig
from tests.util import ellipsoid, f32, rel_l2, smooth_momenta, sym_uniform, uniform

pytestmark = pytest.mark.gpu

INF = float("inf")


def dfs_leaf_order(d):
    """Reference tree (dump) leaf order, children 0..7, bucket members ascending."""
    out = []
    stack = [0]
    ch, leaf, first, nxt = d["children"], d["leaf"], d["first_point"], d["next_point"]
    while stack:
        k = stack.pop()
        if leaf[k]:
            run = []
            i = first[k]
            while i >= 0:
                run.append(i)
                i = nxt[i]
            out.extend(sorted(run))
        else:
            stack.extend(c for c in ch[k][::-1] if c >= 0)
    return np.array(out, np.int32)


def node_multiset(count, amin, amax):
    rows = np.concatenate([count[:, None].astype(np.float64), amin, amax], 1)
    return rows[np.lexsort(rows.T[::-1])]


SETS = {
    "cube": lambda: (uniform(3000, 1.0, 1), sym_uniform(3000, 1.0, 2)),
    "ellipsoid": lambda: (ellipsoid(2500, seed=3), sym_uniform(2500, 0.5, 4)),
    "planar": lambda: (np.stack([np.arange(400) % 20, np.arange(400) // 20, np.zeros(400)], 1) * 1.0,
                       sym_uniform(400, 1.0, 5)),
    "duplicates": lambda: (np.concatenate([np.full((10, 3), 0.5), uniform(990, 2.0, 6)]),
                           sym_uniform(1000, 1.0, 7)),
    # a dense cluster far below the root cell's resolution: long runs of equal
    # 63-bit keys resolved by the deeper digits, plus depth-32 buckets
    "cluster": lambda: (np.concatenate([uniform(3000, 1e-7, 8), np.array([[-1e3, -1e3, -1e3],
                                                                          [1e3, 1e3, 1e3]])]),
                        sym_uniform(3002, 1.0, 9)),
    # sizes with hundreds of radix-sort tiles (decoupled look-back across
    # tiles), with and without neighbours sharing the 63-bit key (the tie check
    # and the full-key fallback sort)
    "cube_200k": lambda: (uniform(200_000, 1.0, 10), sym_uniform(200_000, 1.0, 11)),
    "clusters_120k": lambda: (np.concatenate([uniform(80_000, 1.0, 12)]
                                             + [c + uniform(2_000, 1e-8, 13 + k) for k, c in
                                                enumerate(uniform(20, 1.0, 40))]),
                              sym_uniform(120_000, 1.0, 14)),
    # one run of 12k equal 63-bit keys: k_tie_sort's chunked bitonic sort +
    # three merge passes
    "cluster_12k": lambda: (np.concatenate([uniform(12_000, 1e-7, 15), np.array([[-1e3, -1e3, -1e3],
                                                                                [1e3, 1e3, 1e3]])]),
                            sym_uniform(12_002, 1.0, 16)),
    # the whole cloud in one run (a root box that dwarfs the points, as after a
    # diverged flow): 50 sorted chunks merged over the grid in 6 passes
    "one_run_100k": lambda: (np.concatenate([uniform(100_000, 1.0, 21), np.array([[-1e7, -1e7, -1e7],
                                                                                 [1e7, 1e7, 1e7]])]),
                             sym_uniform(100_002, 1.0, 22)),
    # thousands of short runs (warp-sorted): exact triplicates (ordered by
    # index) and near pairs that differ below level 21 (ordered by key_lo)
    "short_runs": lambda: (lambda b: (np.concatenate([b, b[:100], b[:100], b[100:500] + uniform(400, 1e-8, 18)])[
        np.random.default_rng(19).permutation(6600)], sym_uniform(6600, 1.0, 20)))(uniform(6000, 1.0, 17)),
    "corners": lambda: (np.array([[1.0 if i & 1 else -1.0, 1.0 if i & 2 else -1.0,
                                   1.0 if i & 4 else -1.0] for i in range(8)]), np.zeros((8, 3))),
}


@pytest.mark.parametrize("name", list(SETS))
@pytest.mark.parametrize("prec", [F64, F32])
def test_tree_matches_reference(gs, port, ref, name, prec):
    q, p = SETS[name]()
    if prec == F32:
        q, p = f32(q), f32(p)
    t = gs.build_tree(q, p, precision=prec)
    d = t.download()
    rt = ref.tree(q, p)
    rd = rt.dump()
    # keys: bit-exact vs the oracle's midpoint replay
    kh, kl = port.morton_keys(q)
    assert np.array_equal(d["key_hi"], kh) and np.array_equal(d["key_lo"], kl)
    # leaf order: bit-exact vs the reference octree's DFS
    assert np.array_equal(d["order"], dfs_leaf_order(rd))
    # node set
    assert t.node_count() == rt.node_count()
    assert np.array_equal(node_multiset(d["count"], d["actual_min"], d["actual_max"]),
                          node_multiset(rd["count"], rd["actual_min"], rd["actual_max"]))
    cells = lambda lo, hi: np.concatenate([lo, hi], 1)[np.lexsort(np.concatenate([lo, hi], 1).T[::-1])]
    assert np.array_equal(cells(d["cell_min"], d["cell_max"]), cells(rd["cell_min"], rd["cell_max"]))
    # sums (order-dependent rounding only)
    order = np.lexsort(np.concatenate([d["cell_min"], d["cell_max"]], 1).T[::-1])
    rorder = np.lexsort(np.concatenate([rd["cell_min"], rd["cell_max"]], 1).T[::-1])
    for key in ("position_sum", "momentum_sum"):
        a, b = d[key][order], rd[key][rorder]
        err = np.linalg.norm(a - b, axis=1) / (1.0 + np.linalg.norm(b, axis=1))
        assert err.max() <= 1e-12
    # structural invariants: pre-order, parents, contiguous ranges
    m = t.node_count()
    assert d["parent"][0] == -1 and (d["parent"][1:] < np.arange(1, m)).all()
    assert (d["skip"] > np.arange(m)).all() and d["skip"][0] == m
    assert np.array_equal(d["count"], d["range"][:, 1] - d["range"][:, 0] + 1)


def test_corner_tree_shape(gs):
    q, p = SETS["corners"]()
    t = gs.build_tree(q, p)
    d = t.download()
    assert t.node_count() == 9 and d["count"][0] == 8
    assert (d["level"][1:] == 1).all()


def test_single_point_tree(gs):
    t = gs.build_tree(np.array([[1.0, 2.0, 3.0]]), np.array([[-1.0, 0.5, 0.25]]))
    d = t.download()
    assert t.node_count() == 1 and d["count"][0] == 1
    assert np.array_equal(d["position_sum"][0], [1.0, 2.0, 3.0])
    v, st = t.bh_velocity(np.array([[1.0, 2.0, 3.0]]), 2.0, 1e-9)
    assert np.array_equal(v[0], [-1.0, 0.5, 0.25])
    assert st["direct_interactions"] == 1 and st["approximated_interactions"] == 0


def test_adjoint_accumulation(gs, ref):
    n = 500
    q, p = uniform(n, 5.0, 17), sym_uniform(n, 1.0, 18)
    a, b = sym_uniform(n, 2.0, 19), sym_uniform(n, 2.0, 20)
    t = gs.build_tree(q, p)
    t.accumulate_adjoints(sym_uniform(n, 1.0, 900), sym_uniform(n, 1.0, 901))
    t.accumulate_adjoints(a, b)  # re-annotation overwrites
    d = t.download()
    rt = ref.tree(q, p)
    rt.accumulate(a, b)
    rd = rt.dump()
    o = np.lexsort(np.concatenate([d["cell_min"], d["cell_max"]], 1).T[::-1])
    ro = np.lexsort(np.concatenate([rd["cell_min"], rd["cell_max"]], 1).T[::-1])
    for key in ("alpha_sum", "beta_sum"):
        x, y = d[key][o], rd[key][ro]
        assert (np.linalg.norm(x - y, axis=1) <= 1e-12 * (1 + np.linalg.norm(y, axis=1))).all()


CASES = {
    # name: (q, p, sigma)
    "cube_small_sigma": lambda: (uniform(4000, 1.0, 41), sym_uniform(4000, 1e-2, 42), 0.03),
    "ellipsoid_c2": lambda: (lambda q: (q, smooth_momenta(q, 0.5, 43), 3.0))(ellipsoid(3000, seed=44)),
    "strip": lambda: (np.stack([np.linspace(0, 100, 2000), np.random.default_rng(45).uniform(-2, 2, 2000),
                                np.zeros(2000)], 1), sym_uniform(2000, 1.0, 46), 2.0),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("prec,tol", [(F64, 1e-12), (F32, 1e-5)])
def test_bh_rhs_matches_reference(gs, ref, case, prec, tol):
    q, p, sigma = CASES[case]()
    if prec == F32:
        q, p = f32(q), f32(p)
    thr = 3.0 * sigma
    t = gs.build_tree(q, p, precision=prec)
    dp, dq, st = t.bh_hamiltonian_gradients(sigma, thr)
    per = t.query_stats()
    rt = ref.tree(q, p)
    wp, wq, wper = rt.bh_rhs(sigma, thr, threads=8)
    # the interaction set per query is the reference's, exactly
    assert np.array_equal(per, wper)
    assert st["approximated_interactions"] > 0
    assert rel_l2(dp, wp) <= tol
    assert rel_l2(dq, wq) <= tol


def test_bh_infinite_threshold_is_exact(gs, ref):
    n, sigma = 300, 1.1
    q, p = uniform(n, 8.0, 301), sym_uniform(n, 1.0, 302)
    t = gs.build_tree(q, p)
    dp, dq, st = t.bh_hamiltonian_gradients(sigma, INF)
    wp, wq, _ = ref.exact_rhs(q, p, sigma)
    assert st["approximated_interactions"] == 0 and st["direct_interactions"] == n * n
    assert rel_l2(dp, wp) < 1e-12 and rel_l2(dq, wq) < 1e-12
    h, _ = t.bh_hamiltonian(sigma, INF)
    assert h == pytest.approx(ref.hamiltonian(q, p, sigma), rel=1e-12)


@pytest.mark.parametrize("prec,tol", [(F64, 1e-12), (F32, 2e-5)])
def test_bh_hessian_products_match_reference(gs, ref, prec, tol):
    n, sigma = 3000, 0.05
    q, p = uniform(n, 1.0, 303), sym_uniform(n, 1.0, 304)
    a, b = sym_uniform(n, 1.0, 305), sym_uniform(n, 1.0, 306)
    if prec == F32:
        q, p, a, b = f32(q), f32(p), f32(a), f32(b)
    t = gs.build_tree(q, p, precision=prec)
    t.accumulate_adjoints(a, b)
    *got, st = t.bh_hessian_products(a, b, sigma, 3 * sigma)
    rt = ref.tree(q, p)
    rt.accumulate(a, b)
    want = rt.bh_hessprod(a, b, sigma, 3 * sigma, threads=8)
    assert st["approximated_interactions"] > 0
    for g, w in zip(got, want):
        assert rel_l2(g, w) <= tol


def test_bh_velocity_matches_reference(gs, ref):
    n, sigma = 2000, 0.6
    q, p = uniform(n, 15.0, 61), sym_uniform(n, 1.5, 62)
    x = uniform(500, 15.0, 63)
    t = gs.build_tree(q, p)
    v, st = t.bh_velocity(x, sigma, 3 * sigma)
    rt = ref.tree(q, p)
    wv, wst = rt.bh_velocity(x, sigma, 3 * sigma)
    assert rel_l2(v, wv) <= 1e-12
    assert [st["direct_interactions"], st["approximated_interactions"], st["nodes_visited"]] == \
        list(wst)


@pytest.mark.parametrize("prec,tol", [(F64, 1e-10), (F32, 1e-4)])
def test_bh_shoot_forward_matches_reference(gs, ref, prec, tol):
    n, sigma = 2000, 3.0
    q = ellipsoid(n, seed=71)
    p = smooth_momenta(q, 0.005, 72)  # well-conditioned amplitude
    if prec == F32:
        q, p = f32(q), f32(p)
    cfg = ShootingConfig(sigma=sigma, timesteps=20, backend=BARNES_HUT, precision=prec)
    fq, fp, _, st = gs.shoot_forward(q, p, cfg, keep_trajectory=False)
    wq, wp = ref.shoot_forward(q, p, sigma, 20, backend=1)
    assert rel_l2(fq, wq[-1]) <= tol and rel_l2(fp, wp[-1]) <= tol
    assert st["approximated_interactions"] > 0


@pytest.mark.parametrize("prec,tol", [(F64, 1e-10), (F32, 1e-4)])
def test_bh_evaluate_matches_reference(gs, ref, prec, tol):
    n, sigma = 1500, 2.0
    q = np.stack([np.linspace(0, 100, n), np.random.default_rng(81).uniform(-2, 2, n),
                  np.zeros(n)], 1)
    p = sym_uniform(n, 0.05, 82)
    t = q + np.array([0.0, 0.5, 0.1])
    if prec == F32:
        q, p, t = f32(q), f32(p), f32(t)
    cfg = ShootingConfig(sigma=sigma, lambda_=1.0, timesteps=10, backend=BARNES_HUT, precision=prec)
    ev = gs.evaluate(q, p, t, cfg)
    rep, g, stats, _ = ref.evaluate(q, p, t, sigma, 1.0, 10, 1, threads=8)
    assert ev.report["total"] == pytest.approx(rep[2], rel=tol)
    assert rel_l2(ev.gradient, g) <= tol * 10
    assert ev.stats["approximated_interactions"] > 0


def test_bh_infinite_threshold_evaluate_equals_exact(gs):
    n = 60
    q, p, t = uniform(n, 5.0, 461), sym_uniform(n, 0.3, 462), uniform(n, 5.0, 463)
    a = gs.evaluate(q, p, t, ShootingConfig(sigma=1.2, timesteps=8))
    b = gs.evaluate(q, p, t, ShootingConfig(sigma=1.2, timesteps=8, backend=BARNES_HUT,
                                            threshold_multiplier=INF))
    assert b.report["total"] == pytest.approx(a.report["total"], rel=1e-10)
    assert rel_l2(b.gradient, a.gradient) < 1e-10


def test_bh_rk4_matches_composed_oracle(gs, port):
    n, sigma = 3000, 0.03
    q = uniform(n, 1.0, 91)
    p = np.random.default_rng(92).normal(0, 1e-4, (n, 3))
    cfg = ShootingConfig(sigma=sigma, timesteps=5, backend=BARNES_HUT, integrator=RK4)
    fq, fp, _, _ = gs.shoot_forward(q, p, cfg, keep_trajectory=False)
    w = port.shoot_forward(q, p, sigma, 5, backend=1, integrator=1, keep_traj=False)
    assert rel_l2(fq, w["q"]) <= 1e-10 and rel_l2(fp, w["p"]) <= 1e-10


def test_bh_warp_carrier_points(gs):
    n = 20
    q, p = uniform(n, 1.5, 471), sym_uniform(n, 0.25, 472)
    cfg = ShootingConfig(sigma=0.8, timesteps=20, backend=BARNES_HUT)
    tr = gs.shoot_forward(q, p, cfg)
    warped = gs.warp_points(tr, q, cfg)
    assert np.abs(warped - tr.q[-1]).max() < 1e-10


# ---- literal-mean-dot mode: pinned to the reference built with
# GEOSHOOT_BH_LITERAL_MEAN_DOT (oracle/_ref/libgeoshoot_ref_lmd.so) ----------
@pytest.fixture
def ref_lmd():
    import oracle
    if not os.path.exists(oracle.REF_LMD_SO):
        pytest.skip("oracle/_ref/libgeoshoot_ref_lmd.so not built")
    return oracle.ref_lmd()


@pytest.fixture
def gs_lmd(gs):
    gs.set_literal_mean_dot(True)
    yield gs
    gs.set_literal_mean_dot(False)


@pytest.mark.parametrize("prec,tol", [(F64, 1e-12), (F32, 1e-5)])
def test_lmd_tree_calls_match_reference(gs_lmd, ref, ref_lmd, prec, tol):
    gs = gs_lmd
    q, p, sigma = CASES["cube_small_sigma"]()
    a, b = sym_uniform(len(q), 1.0, 991), sym_uniform(len(q), 1.0, 992)
    if prec == F32:
        q, p, a, b = f32(q), f32(p), f32(a), f32(b)
    thr = 3.0 * sigma
    t = gs.build_tree(q, p, precision=prec)
    dp, dq, st = t.bh_hamiltonian_gradients(sigma, thr)
    rt = ref_lmd.tree(q, p)
    wp, wq, wper = rt.bh_rhs(sigma, thr, threads=8)
    assert np.array_equal(t.query_stats(), wper)
    assert rel_l2(dp, wp) <= tol and rel_l2(dq, wq) <= tol
    # the scale changes dH/dq (and only it) against the default build
    _, dq0, _ = ref.tree(q, p).bh_rhs(sigma, thr, threads=8)
    assert rel_l2(dq, dq0) > 100 * tol
    h, _ = t.bh_hamiltonian(sigma, thr)
    assert h == pytest.approx(rt.bh_hamiltonian(sigma, thr), rel=tol)
    t.accumulate_adjoints(a, b)
    *got, _ = t.bh_hessian_products(a, b, sigma, thr)
    rt.accumulate(a, b)
    want = rt.bh_hessprod(a, b, sigma, thr, threads=8)
    for g, w in zip(got, want):
        assert rel_l2(g, w) <= 2 * tol


@pytest.mark.parametrize("prec,tol", [(F64, 1e-10), (F32, 1e-4)])
def test_lmd_shooting_matches_reference(gs, ref_lmd, prec, tol):
    n, sigma = 1500, 2.0
    q = np.stack([np.linspace(0, 100, n), np.random.default_rng(83).uniform(-2, 2, n),
                  np.zeros(n)], 1)
    p = sym_uniform(n, 0.05, 84)
    t = q + np.array([0.0, 0.5, 0.1])
    if prec == F32:
        q, p, t = f32(q), f32(p), f32(t)
    cfg = ShootingConfig(sigma=sigma, lambda_=1.0, timesteps=10, backend=BARNES_HUT, precision=prec,
                         literal_mean_dot=True)
    fq, fp, _, _ = gs.shoot_forward(q, p, cfg, keep_trajectory=False)
    wq, wp = ref_lmd.shoot_forward(q, p, sigma, 10, backend=1)
    assert rel_l2(fq, wq[-1]) <= tol and rel_l2(fp, wp[-1]) <= tol
    ev = gs.evaluate(q, p, t, cfg)
    rep, g, _, _ = ref_lmd.evaluate(q, p, t, sigma, 1.0, 10, 1, threads=8)
    assert ev.report["total"] == pytest.approx(rep[2], rel=tol)
    assert rel_l2(ev.gradient, g) <= tol * 10


REPLAY = r"""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_1907_04834_b200 import Geoshoot, F32, F64
from tests.test_gpu_bh import SETS, dfs_leaf_order
import oracle
gs, ref = Geoshoot(0), oracle.ref()
for name in ("duplicates", "cluster", "clusters_120k", "cluster_12k", "short_runs", "one_run_100k"):
    for prec in (F64, F32):
        q, p = SETS[name]()
        if prec == F32:
            q, p = q.astype(np.float32).astype(np.float64), p.astype(np.float32).astype(np.float64)
        d = gs.build_tree(q, p, precision=prec).download()
        assert np.array_equal(d["order"], dfs_leaf_order(ref.tree(q, p).dump())), (name, prec)
print("ok")
"""


def test_tie_sort_replays_the_deep_key():
    """k_keys computes the deep key only when the previous build of the tree had
    ties; otherwise the tie sort replays it for the run members. GS_KEYS_LO=0
    forces the replay for every build: the leaf order must still be the
    reference's on every tie set."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", REPLAY], cwd=root, capture_output=True, text=True,
                       timeout=900, env=dict(os.environ, GS_KEYS_LO="0"))
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]
