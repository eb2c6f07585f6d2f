"""Every Barnes-Hut walk and node-window split against the reference.

The device has three walks over the same pre-order node records -- independent
per-lane walks (k_bh_ws), the group walk (k_bh_grp, default for dense near
fields) and a split launch by warp query box -- and splits the node array into
K windows for occupancy (bh_tasks). Whatever the choice, each query's
interaction set must be the reference's (traverse, bh_kernel.cpp:30-58): the
per-query (direct, approximated, visited) counts -- folded over the windows --
are asserted EQUAL to oracle/_ref's, and the values to FP64 1e-12 / FP32 1e-5
(FP32-rounded inputs). gs_set_bh_walk forces the walk; kernel 0 / windows 0 is
the production choice by regime.

Also: bh_point_gradients / bh_point_hessian_products (bh_kernel.cpp:81-160) at
ARBITRARY query points (tree points or not), with per-point adjoints that
differ from the tree's annotation, through the same walks.
"""
import numpy as np
import pytest

from paper_1907_04834_b200 import F32, F64
from tests.util import ellipsoid, f32, rel_l2, smooth_momenta, sym_uniform, uniform

pytestmark = pytest.mark.gpu

CASES = {
    # sparse near field (config 4 regime): independent walks by default
    "cube_sparse": lambda: (uniform(4000, 1.0, 41), sym_uniform(4000, 1e-2, 42), 0.03),
    # config 2 at full size: thousands of points within 3 sigma -> dense regime
    # (group walk, 32 windows by default)
    "c2_ellipsoid_20k": lambda: (lambda q: (q, smooth_momenta(q, 0.5, 43), 3.0))(
        ellipsoid(20000, seed=44)),
    # elongated: long thin near fields
    "strip": lambda: (np.stack([np.linspace(0, 100, 2000),
                                np.random.default_rng(45).uniform(-2, 2, 2000),
                                np.zeros(2000)], 1), sym_uniform(2000, 1.0, 46), 2.0),
}
KERNELS = [0, 1, 3, 4]   # by regime, independent, group, split
WINDOWS = [0, 1, 7, 32]  # automatic, or K windows
TOL = {F64: 1e-12, F32: 1e-5}

_cache = {}


def case_data(name, prec):
    key = (name, prec)
    if key not in _cache:
        q, p, sigma = CASES[name]()
        if prec == F32:
            q, p = f32(q), f32(p)
        n = len(q)
        a, b = sym_uniform(n, 1.0, 501), sym_uniform(n, 1.0, 502)
        if prec == F32:
            a, b = f32(a), f32(b)
        _cache[key] = dict(q=q, p=p, sigma=sigma, a=a, b=b)
    return _cache[key]


_ref_cache = {}


def ref_results(ref, name, prec, what):
    key = (name, prec, what)
    if key not in _ref_cache:
        d = case_data(name, prec)
        rt = ref.tree(d["q"], d["p"])
        thr = 3.0 * d["sigma"]
        if what == "rhs":
            _ref_cache[key] = rt.bh_rhs(d["sigma"], thr, threads=0)
        else:
            rt.accumulate(d["a"], d["b"])
            _ref_cache[key] = rt.bh_hessprod(d["a"], d["b"], d["sigma"], thr, threads=0,
                                             per_query=True)
    return _ref_cache[key]


@pytest.fixture
def walk(gs):
    def set_walk(kernel, windows):
        gs.set_bh_walk(kernel, windows)
    yield set_walk
    gs.set_bh_walk(-1, -1)


@pytest.mark.parametrize("windows", WINDOWS)
@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("prec", [F64, F32])
@pytest.mark.parametrize("name", list(CASES))
def test_walk_rhs_matches_reference(gs, ref, walk, name, prec, kernel, windows):
    d = case_data(name, prec)
    walk(kernel, windows)
    t = gs.build_tree(d["q"], d["p"], precision=prec)
    dp, dq, st = t.bh_hamiltonian_gradients(d["sigma"], 3.0 * d["sigma"])
    per = t.query_stats()
    wp, wq, wper = ref_results(ref, name, prec, "rhs")
    assert np.array_equal(per, wper), np.argwhere((per != wper).any(1))[:5]
    assert st["approximated_interactions"] == int(wper[:, 1].sum()) > 0
    assert st["direct_interactions"] == int(wper[:, 0].sum())
    assert st["nodes_visited"] == int(wper[:, 2].sum())
    assert rel_l2(dp, wp) <= TOL[prec] and rel_l2(dq, wq) <= TOL[prec]


@pytest.mark.parametrize("windows", [1, 7, 32])
@pytest.mark.parametrize("kernel", [1, 3, 4])
@pytest.mark.parametrize("prec", [F64, F32])
@pytest.mark.parametrize("name", ["cube_sparse", "c2_ellipsoid_20k"])
def test_walk_hessprod_matches_reference(gs, ref, walk, name, prec, kernel, windows):
    d = case_data(name, prec)
    walk(kernel, windows)
    t = gs.build_tree(d["q"], d["p"], precision=prec)
    t.accumulate_adjoints(d["a"], d["b"])
    *got, st = t.bh_hessian_products(d["a"], d["b"], d["sigma"], 3.0 * d["sigma"])
    per = t.query_stats()
    *want, wper = ref_results(ref, name, prec, "hess")
    assert np.array_equal(per, wper)
    assert st["approximated_interactions"] > 0
    for g, w in zip(got, want):
        assert rel_l2(g, w) <= 2 * TOL[prec]


@pytest.mark.parametrize("windows", [0, 1, 7, 32])
@pytest.mark.parametrize("kernel", [0, 1, 3, 4])
def test_walk_velocity_matches_reference(gs, ref, walk, kernel, windows):
    d = case_data("c2_ellipsoid_20k", F64)
    x = np.concatenate([d["q"][::7], ellipsoid(1500, seed=77), uniform(200, 80.0, 78) - 40.0])
    walk(kernel, windows)
    t = gs.build_tree(d["q"], d["p"])
    v, st = t.bh_velocity(x, d["sigma"], 3.0 * d["sigma"])
    per = t.query_stats()
    rt = ref.tree(d["q"], d["p"])
    wv, wper = rt.bh_velocity_pq(x, d["sigma"], 3.0 * d["sigma"])
    assert np.array_equal(per, wper)
    assert rel_l2(v, wv) <= 1e-12


def query_points(d, seed):
    """Tree points, their neighbours, and points far outside the cloud."""
    q = d["q"]
    rng = np.random.default_rng(seed)
    pick = rng.choice(len(q), 300, replace=False)
    ext = q.max(0) - q.min(0)
    x = np.concatenate([q[pick[:100]],
                        q[pick[100:250]] + rng.normal(0, 0.3 * d["sigma"], (150, 3)),
                        q.min(0) + rng.uniform(-0.5, 1.5, (50, 3)) * ext])
    px = np.concatenate([d["p"][pick[:100]], sym_uniform(200, 0.5, seed + 1)])
    return x, px


@pytest.mark.parametrize("kernel,windows", [(0, 0), (1, 1), (3, 7), (4, 32)])
@pytest.mark.parametrize("prec", [F64, F32])
@pytest.mark.parametrize("name", ["cube_sparse", "c2_ellipsoid_20k"])
def test_point_gradients_arbitrary_queries(gs, ref, walk, name, prec, kernel, windows):
    d = case_data(name, prec)
    x, px = query_points(d, 600)
    if prec == F32:
        x, px = f32(x), f32(px)
    walk(kernel, windows)
    t = gs.build_tree(d["q"], d["p"], precision=prec)
    dp, dq, st = t.bh_point_gradients(x, px, d["sigma"], 3.0 * d["sigma"])
    per = t.query_stats()
    rt = ref.tree(d["q"], d["p"])
    wp, wq, wper = rt.bh_point_gradients(x, px, d["sigma"], 3.0 * d["sigma"])
    assert np.array_equal(per, wper)
    assert st["direct_interactions"] == int(wper[:, 0].sum())
    assert rel_l2(dp, wp) <= TOL[prec] and rel_l2(dq, wq) <= TOL[prec]


@pytest.mark.parametrize("kernel,windows", [(0, 0), (1, 1), (3, 7), (4, 32)])
@pytest.mark.parametrize("prec", [F64, F32])
@pytest.mark.parametrize("name", ["cube_sparse", "c2_ellipsoid_20k"])
def test_point_hessprod_arbitrary_queries(gs, ref, walk, name, prec, kernel, windows):
    """alpha_i / beta_i are independent inputs, and the direct terms' per-point
    adjoints differ from the tree's annotation (node sums): the reference reads
    the passed arrays for direct terms and the node sums for approximated ones."""
    d = case_data(name, prec)
    x, px = query_points(d, 700)
    n, m = len(d["q"]), len(x)
    ai, bi = sym_uniform(m, 1.0, 701), sym_uniform(m, 1.0, 702)
    a2, b2 = sym_uniform(n, 1.0, 703), sym_uniform(n, 1.0, 704)
    if prec == F32:
        x, px, ai, bi, a2, b2 = (f32(v) for v in (x, px, ai, bi, a2, b2))
    walk(kernel, windows)
    t = gs.build_tree(d["q"], d["p"], precision=prec)
    t.accumulate_adjoints(d["a"], d["b"])
    *got, st = t.bh_point_hessian_products(x, px, ai, bi, a2, b2, d["sigma"], 3.0 * d["sigma"])
    per = t.query_stats()
    rt = ref.tree(d["q"], d["p"])
    rt.accumulate(d["a"], d["b"])
    *want, wper = rt.bh_point_hessprod(x, px, ai, bi, a2, b2, d["sigma"], 3.0 * d["sigma"])
    assert np.array_equal(per, wper)
    for g, w in zip(got, want):
        assert rel_l2(g, w) <= 2 * TOL[prec]
    # alpha = beta = None: the per-point adjoints of the last upload (a2, b2) stay
    *again, _ = t.bh_point_hessian_products(x, px, ai, bi, None, None, d["sigma"],
                                            3.0 * d["sigma"])
    for g, h in zip(got, again):
        assert np.array_equal(g, h)


def test_point_hessprod_without_annotation_uses_zero_node_sums(gs, ref):
    d = case_data("cube_sparse", F64)
    x, px = query_points(d, 800)
    m = len(x)
    ai, bi = sym_uniform(m, 1.0, 801), sym_uniform(m, 1.0, 802)
    t = gs.build_tree(d["q"], d["p"])
    *got, _ = t.bh_point_hessian_products(x, px, ai, bi, d["a"], d["b"], d["sigma"],
                                          3.0 * d["sigma"])
    rt = ref.tree(d["q"], d["p"])  # never annotated: Node sums are zero
    *want, _ = rt.bh_point_hessprod(x, px, ai, bi, d["a"], d["b"], d["sigma"], 3.0 * d["sigma"])
    for g, w in zip(got, want):
        assert rel_l2(g, w) <= 1e-12


def test_walk_choice_is_validated(gs):
    with pytest.raises(ValueError):
        gs.set_bh_walk(2, 0)
    with pytest.raises(ValueError):
        gs.set_bh_walk(1, 65)
    gs.set_bh_walk(-1, -1)
