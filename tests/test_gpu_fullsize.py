"""Full-size (BASELINE config 4: N = 1,000,000, unit cube, sigma = 0.0131)
checks through size-independent properties, where the oracle cannot run the
whole problem in test time:

* exact RHS: a random sample of targets against an FP64 numpy restatement of
  kernel_exact.cpp:29-61 over ALL 1M sources; Newton's third law
  (sum_i dH/dq_i = 0: the pair terms are antisymmetric); bitwise determinism;
* Barnes-Hut: every query accounts for every point exactly once -- with
  p = e_x and sigma so large that G == 1.0f exactly, dH/dp_i = 2 sum over the
  query's units of (point count) must be exactly 2N for all 1M queries, at a
  threshold that mixes direct and approximated units; the tree is a valid
  pre-order Morton tree (sorted keys, nested ranges, counts).
"""
import numpy as np
import pytest

from paper_1907_04834_b200 import F32, F64
from tests.util import f32

pytestmark = pytest.mark.gpu

N = 1_000_000
SIGMA = 0.0131


def cube(n=N, seed=2024):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.0, 1.0, (n, 3)), rng.normal(0.0, 1e-2, (n, 3))


def oracle_rows(q, p, rows, sigma):
    """FP64 restatement of hamiltonian_with_gradients for the given targets."""
    inv_two_s, two_over_s = 1.0 / (2 * sigma * sigma), 2.0 / (sigma * sigma)
    dp = np.empty((len(rows), 3))
    dq = np.empty((len(rows), 3))
    for k, i in enumerate(rows):
        d = q[i] - q
        g = np.exp(-(d * d).sum(1) * inv_two_s)
        dp[k] = 2.0 * (g[:, None] * p).sum(0)
        c = (p @ p[i]) * g
        dq[k] = -two_over_s * (c[:, None] * d).sum(0)
    return dp, dq


def test_exact_rhs_full_size(gs):
    q, p = cube()
    q, p = f32(q), f32(p)
    _, dp, dq = gs.hamiltonian_with_gradients(q, p, SIGMA, precision=F32)
    rows = np.random.default_rng(7).choice(N, 48, replace=False)
    wp, wq = oracle_rows(q, p, rows, SIGMA)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    assert rel(dp[rows], wp) < 1e-5
    assert rel(dq[rows], wq) < 1e-5
    # pair terms are antisymmetric: the total "force" vanishes
    assert np.linalg.norm(dq.sum(0)) <= 1e-5 * np.abs(dq).sum()
    _, dp2, dq2 = gs.hamiltonian_with_gradients(q, p, SIGMA, precision=F32)
    assert np.array_equal(dp, dp2) and np.array_equal(dq, dq2)


@pytest.mark.parametrize("prec", [F32, F64])
def test_bh_full_size_covers_every_point_once(gs, prec):
    q, _ = cube(seed=11)
    if prec == F32:
        q = f32(q)
    p = np.zeros_like(q)
    p[:, 0] = 1.0
    t = gs.build_tree(q, p, precision=prec)
    big_sigma, thr = 1e6, 0.03  # G == 1 for every unit; the gate still mixes units
    dp, _, st = t.bh_hamiltonian_gradients(big_sigma, thr)
    assert st["approximated_interactions"] > 10 * N and st["direct_interactions"] > 10 * N
    if prec == F32:
        assert (dp[:, 0] == 2.0 * N).all() and (dp[:, 1:] == 0).all()
    else:
        assert np.abs(dp[:, 0] / (2.0 * N) - 1.0).max() < 1e-9
    per = t.query_stats()
    assert (per[:, 0] + per[:, 1] >= 1).all() and (per[:, 2] >= 1).all()
    d = t.download()
    keys = d["key_hi"][d["order"]]
    assert (keys[1:] >= keys[:-1]).all()  # leaf order is Morton order
    m = t.node_count()
    assert d["skip"][0] == m and (d["skip"] > np.arange(m)).all()
    assert d["count"][0] == N
    assert np.array_equal(d["count"], d["range"][:, 1] - d["range"][:, 0] + 1)


def test_bh_infinite_threshold_equals_exact_config2_fp64(gs):
    """Config 2 size (N = 20k ellipsoid, sigma 3, 20 Euler steps, FP64): with an
    infinite gate every unit is direct, so Barnes-Hut must reproduce the exact
    flow (the reference's own property, test_bh_kernel.cpp:58-110, here at the
    config's full size)."""
    from paper_1907_04834_b200 import BARNES_HUT, EXACT, ShootingConfig
    from tests.util import ellipsoid, rel_l2, smooth_momenta
    q = ellipsoid(20000, seed=44)
    p = smooth_momenta(q, 0.005, 43)
    base = dict(sigma=3.0, timesteps=20, precision=F64)
    eq, ep, ee, _ = gs.shoot_forward(q, p, ShootingConfig(backend=EXACT, **base),
                                     keep_trajectory=False)
    bq, bp, be, st = gs.shoot_forward(
        q, p, ShootingConfig(backend=BARNES_HUT, threshold_multiplier=float("inf"), **base),
        keep_trajectory=False)
    assert st["approximated_interactions"] == 0
    assert st["direct_interactions"] == 20 * 20000 ** 2
    assert rel_l2(bq, eq) < 1e-12 and rel_l2(bp, ep) < 1e-10
    assert be == pytest.approx(ee, rel=1e-12)


def test_bh_infinite_threshold_equals_exact_config3_evaluate(gs):
    """Config 3 size (N = 50k tube, sigma 5, T = 20, FP32): the fused forward +
    adjoint evaluate() through the tree with an infinite gate equals the exact
    evaluate() (objective and gradient)."""
    from paper_1907_04834_b200 import BARNES_HUT, EXACT, ShootingConfig
    from tests.util import rel_l2, smooth_momenta, tube
    q = f32(tube(50000, seed=3))
    p = f32(smooth_momenta(q, 0.01, 4))
    t = f32(q + 0.05)
    base = dict(sigma=5.0, lambda_=100.0, timesteps=20, precision=F32)
    a = gs.evaluate(q, p, t, ShootingConfig(backend=EXACT, **base))
    b = gs.evaluate(q, p, t, ShootingConfig(backend=BARNES_HUT, threshold_multiplier=float("inf"),
                                            **base))
    assert b.stats["approximated_interactions"] == 0
    assert b.report["total"] == pytest.approx(a.report["total"], rel=1e-5)
    assert rel_l2(b.gradient, a.gradient) < 1e-4
