"""Per-RHS parity against the reference (oracle/_ref) at BASELINE.json's full
configuration sizes, through the production walk choice (gs_set_bh_walk
untouched: group walk + 32 node windows in the dense configs 2/3/5,
independent walks in the sparse config 4).

Each case builds the config's point set with the seeded generators of
tests/util.py (FP32 runs get FP32-rounded inputs), runs ONE
Barnes-Hut right-hand side (bh_hamiltonian_gradients, bh_kernel.cpp:193-210)
and, where noted, one Hessian-product pass (bh_hessian_products :212-236) on
the B200, and asserts

* per-query (direct, approximated, visited) counts EQUAL to the reference's
  per-query TraversalStats (integer work: bit-exact),
* values to FP64 1e-12 / FP32 1e-5 relative L2 (per-RHS tolerance).

The exact path at config 4's N = 1M is pinned the same way: dH/dp = 2 v
(kernel_exact.hpp:22-28) on sampled targets against the reference's own
exact_velocity (kernel_exact.cpp:70-82) over all 1M sources.
"""
import numpy as np
import pytest

from paper_1907_04834_b200 import F32, F64
from tests.util import ellipsoid, f32, rel_l2, smooth_momenta, sym_uniform, tube

pytestmark = pytest.mark.gpu

TOL = {F64: 1e-12, F32: 1e-5}


def c2(prec):
    q = ellipsoid(20000, seed=2)
    return q, smooth_momenta(q, 0.5, 3), 3.0


def c3_template(prec):
    q = tube(50000, seed=5)
    return q, smooth_momenta(q, 1.0, 6), 5.0


def c4(n):
    def make(prec):
        rng = np.random.default_rng(2024 + n)
        return rng.uniform(0.0, 1.0, (n, 3)), rng.normal(0.0, 1e-2, (n, 3)), 0.0131
    return make


def c5_subject(prec, k=0):
    rng = np.random.default_rng(5000 + k)
    axes = (rng.uniform(25, 35), rng.uniform(12, 18), rng.uniform(8, 12))
    q = ellipsoid(30000, axes=axes, seed=5100 + k)
    return q, smooth_momenta(q, 0.8, 5200 + k), 3.0


CASES = {
    "c2_20k_fp64": (c2, F64),
    "c2_20k_fp32": (c2, F32),
    "c3_50k_fp32": (c3_template, F32),
    "c4_100k_fp32": (c4(100_000), F32),
    "c4_1m_fp32": (c4(1_000_000), F32),
    "c5_30k_fp32": (c5_subject, F32),
}


@pytest.mark.parametrize("name", list(CASES))
def test_bh_rhs_at_baseline_size(gs, ref, name):
    make, prec = CASES[name]
    q, p, sigma = make(prec)
    if prec == F32:
        q, p = f32(q), f32(p)
    thr = 3.0 * sigma
    t = gs.build_tree(q, p, precision=prec)
    dp, dq, st = t.bh_hamiltonian_gradients(sigma, thr)
    per = t.query_stats()
    rt = ref.tree(q, p)
    wp, wq, wper = rt.bh_rhs(sigma, thr, threads=0)
    bad = np.argwhere((per != wper).any(1))[:, 0]
    assert bad.size == 0, (bad[:5], per[bad[:5]], wper[bad[:5]])
    assert st["approximated_interactions"] > 0
    assert rel_l2(dp, wp) <= TOL[prec]
    assert rel_l2(dq, wq) <= TOL[prec]


@pytest.mark.parametrize("name", ["c2_20k_fp64", "c2_20k_fp32", "c5_30k_fp32"])
def test_bh_hessprod_at_baseline_size(gs, ref, name):
    make, prec = CASES[name]
    q, p, sigma = make(prec)
    n = len(q)
    a, b = sym_uniform(n, 1.0, 91), sym_uniform(n, 1.0, 92)
    if prec == F32:
        q, p, a, b = f32(q), f32(p), f32(a), f32(b)
    thr = 3.0 * sigma
    t = gs.build_tree(q, p, precision=prec)
    t.accumulate_adjoints(a, b)
    *got, st = t.bh_hessian_products(a, b, sigma, thr)
    per = t.query_stats()
    rt = ref.tree(q, p)
    rt.accumulate(a, b)
    *want, wper = rt.bh_hessprod(a, b, sigma, thr, threads=0, per_query=True)
    assert np.array_equal(per, wper)
    for g, w in zip(got, want):
        assert rel_l2(g, w) <= 2 * TOL[prec]


def test_exact_dhdp_1m_against_reference_velocity(gs, ref):
    """Config 4 exact RHS at N = 1M (FP32): dH/dp_i = 2 sum_j G_ij p_j = 2 v(q_i)
    against the reference's exact_velocity over all 1M sources, FP64."""
    q, p, sigma = c4(1_000_000)(F32)
    q, p = f32(q), f32(p)
    _, dp, _ = gs.hamiltonian_with_gradients(q, p, sigma, precision=F32)
    rows = np.random.default_rng(8).choice(len(q), 48, replace=False)
    v = ref.exact_velocity(q[rows], q, p, sigma)
    assert rel_l2(dp[rows], 2.0 * v) < 1e-5


def test_exact_f64_dhdp_1m_against_reference_velocity(gs, ref):
    """Config 4 exact RHS at N = 1M in FP64 (the symmetric FP64 kernel, 977
    tiles, diagonals in 16 groups): dH/dp = 2 v on sampled targets against the
    reference's exact_velocity over all 1M sources."""
    q, p, sigma = c4(1_000_000)(F64)
    assert gs.exact_pairs_plan(len(q), F64) > 0
    _, dp, _ = gs.hamiltonian_with_gradients(q, p, sigma, precision=F64)
    rows = np.random.default_rng(9).choice(len(q), 32, replace=False)
    v = ref.exact_velocity(q[rows], q, p, sigma)
    assert rel_l2(dp[rows], 2.0 * v) < 1e-12


def test_exact_adjoint_c3_symmetric_equals_gather(gs):
    """Config 3 size (50k tube): the symmetric Hessian-product kernel against
    the gather kernel (each checked against the reference at small N in
    test_gpu_exact.py) -- FP32 rounding apart."""
    q, p, sigma = c3_template(F32)
    q, p = f32(q), f32(p)
    n = len(q)
    a, b = f32(sym_uniform(n, 1.0, 93)), f32(sym_uniform(n, 1.0, 94))
    assert gs.exact_pairs_plan(n, F32) > 0
    sym = gs.hessian_products(q, p, a, b, sigma, precision=F32)
    gs.set_exact_pairs(1)
    try:
        gather = gs.hessian_products(q, p, a, b, sigma, precision=F32)
    finally:
        gs.set_exact_pairs(-1)
    for s_, g_ in zip(sym, gather):
        assert rel_l2(s_, g_) < 2e-6
