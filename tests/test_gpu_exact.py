"""Parity of the exact (all-pairs) CUDA path against the reference oracle.

Tolerances (BASELINE.json north_star): FP64 relative L2 <= 1e-10 on final q
and p; FP32 <= 1e-4 (per RHS we hold FP32 to 1e-5, the FP32-input floor being
~1e-6). FP32 runs compare against the oracle given the same
FP32-rounded inputs.
"""
import numpy as np
import pytest

from paper_1907_04834_b200 import (EXACT, F32, F64, RK4, ConfigError, ConfigMismatch,
                                   DimensionMismatch, NonFiniteState, ShootingConfig)
from tests.util import f32, rel_l2, sphere, sym_uniform, uniform

pytestmark = pytest.mark.gpu

F64_TOL = 1e-10
F32_RHS_TOL = 1e-5
F32_TRAJ_TOL = 1e-4


# ---------------------------------------------------------------- kernel_exact
@pytest.mark.parametrize("n", [1, 3, 127, 1000, 4099])
def test_exact_rhs_f64_matches_reference(gs, ref, n):
    q, p = uniform(n, 8.0, seed=n), sym_uniform(n, 1.0, seed=n + 1)
    h, dp, dq = gs.hamiltonian_with_gradients(q, p, 1.1)
    wp, wq, wh = ref.exact_rhs(q, p, 1.1)
    assert rel_l2(dp, wp) < 1e-13
    assert rel_l2(dq, wq) < 1e-12 or np.abs(dq - wq).max() < 1e-14
    assert abs(h - wh) <= 1e-12 * abs(wh)


@pytest.mark.parametrize("n", [5, 1000, 4099])
def test_exact_rhs_f32_matches_reference(gs, ref, n):
    q, p = f32(uniform(n, 8.0, seed=n)), f32(sym_uniform(n, 1.0, seed=n + 1))
    h, dp, dq = gs.hamiltonian_with_gradients(q, p, 1.1, precision=F32)
    wp, wq, wh = ref.exact_rhs(q, p, 1.1)
    assert rel_l2(dp, wp) < F32_RHS_TOL
    assert rel_l2(dq, wq) < F32_RHS_TOL
    assert abs(h - wh) <= F32_RHS_TOL * abs(wh)


def test_known_answers(gs):
    # single point: H = |p|^2, dH/dp = 2p exactly, dH/dq = 0 (test_kernel_exact.cpp:65-69,136-142)
    q = np.array([[1.0, 2.0, 3.0]])
    p = np.array([[0.5, -1.0, 0.25]])
    h, dp, dq = gs.hamiltonian_with_gradients(q, p, 3.0)
    assert np.array_equal(dp, 2 * p) and np.array_equal(dq, np.zeros((1, 3)))
    assert h == pytest.approx(1.3125, rel=1e-15)
    # zero momentum -> zero field and zero gradients
    q = uniform(6, 5.0, 11)
    h, dp, dq = gs.hamiltonian_with_gradients(q, np.zeros((6, 3)), 1.5)
    assert h == 0.0 and not dp.any() and not dq.any()


def test_flow_factor_two(gs, ref):
    # dH/dp == 2 * exact_velocity (kernel_exact.hpp:22-28, test_kernel_exact.cpp:190-200)
    q, p = uniform(8, 3.0, 81), sym_uniform(8, 1.0, 82)
    dp, _ = gs.hamiltonian_gradients(q, p, 1.4)
    v = gs.exact_velocity(q, q, p, 1.4)
    assert np.allclose(dp, 2.0 * v, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("prec,tol", [(F64, 1e-13), (F32, F32_RHS_TOL)])
def test_exact_velocity_matches_reference(gs, ref, prec, tol):
    q, p = uniform(700, 3.0, 71), sym_uniform(700, 1.5, 72)
    x = uniform(333, 3.0, 73)
    if prec == F32:
        q, p, x = f32(q), f32(p), f32(x)
    v = gs.exact_velocity(x, q, p, 0.4, precision=prec)
    assert rel_l2(v, ref.exact_velocity(x, q, p, 0.4)) < tol


@pytest.mark.parametrize("prec,tol", [(F64, 1e-12), (F32, 2e-5)])
@pytest.mark.parametrize("n", [4, 600])
def test_hessian_products_match_reference(gs, ref, prec, tol, n):
    q, p = uniform(n, 2.0 + n / 100, 91), sym_uniform(n, 1.0, 92)
    a, b = sym_uniform(n, 1.0, 93), sym_uniform(n, 1.0, 94)
    if prec == F32:
        q, p, a, b = f32(q), f32(p), f32(a), f32(b)
    got = gs.hessian_products(q, p, a, b, 1.2, precision=prec)
    want = ref.hessian_products(q, p, a, b, 1.2)
    for g, w in zip(got, want):
        assert rel_l2(g, w) < tol


def test_dimension_mismatch(gs):
    with pytest.raises(DimensionMismatch):
        gs.hamiltonian(uniform(3, 1.0, 1), np.zeros((4, 3)), 1.0)


# ---------------------------------------------------------------- shooting
def c1_inputs(n=1024, seed=7):
    q = sphere(n, seed)
    p = np.random.default_rng(seed + 1).normal(0, 0.01, (n, 3))
    return q, p


def test_config1_exact_f64(gs, ref):
    """BASELINE config 1: N=1024 unit sphere, sigma 0.2, 10 Euler steps, FP64."""
    q, p = c1_inputs()
    cfg = ShootingConfig(sigma=0.2, timesteps=10, backend=EXACT, precision=F64)
    tr = gs.shoot_forward(q, p, cfg)
    wq, wp = ref.shoot_forward(q, p, 0.2, 10)
    assert rel_l2(tr.q[-1], wq[-1]) <= F64_TOL
    assert rel_l2(tr.p[-1], wp[-1]) <= F64_TOL
    assert rel_l2(tr.q, wq) <= F64_TOL
    fq, fp, energy, _ = gs.shoot_forward(q, p, cfg, keep_trajectory=False)
    assert np.array_equal(fq, tr.q[-1]) and np.array_equal(fp, tr.p[-1])
    assert energy == pytest.approx(ref.hamiltonian(q, p, 0.2), rel=1e-12)


def test_config1_exact_f32(gs, ref):
    q, p = c1_inputs()
    q, p = f32(q), f32(p)
    cfg = ShootingConfig(sigma=0.2, timesteps=10, backend=EXACT, precision=F32)
    fq, fp, _, _ = gs.shoot_forward(q, p, cfg, keep_trajectory=False)
    wq, wp = ref.shoot_forward(q, p, 0.2, 10)
    assert rel_l2(fq, wq[-1]) <= F32_TRAJ_TOL
    assert rel_l2(fp, wp[-1]) <= F32_TRAJ_TOL


@pytest.mark.parametrize("prec,tol", [(F64, F64_TOL), (F32, F32_TRAJ_TOL)])
def test_rk4_matches_composed_oracle(gs, port, prec, tol):
    """RK4 (BASELINE config 4) against the CPU RK4 composed over the reference RHS."""
    n = 800
    q = uniform(n, 1.0, 31)
    p = np.random.default_rng(32).normal(0, 1e-2, (n, 3))
    if prec == F32:
        q, p = f32(q), f32(p)
    cfg = ShootingConfig(sigma=0.05, timesteps=10, backend=EXACT, integrator=RK4, precision=prec)
    fq, fp, e, _ = gs.shoot_forward(q, p, cfg, keep_trajectory=False)
    w = port.shoot_forward(q, p, 0.05, 10, integrator=1, keep_traj=False)
    assert rel_l2(fq, w["q"]) <= tol
    assert rel_l2(fp, w["p"]) <= tol
    assert e == pytest.approx(w["energy"], rel=1e-12 if prec == F64 else 1e-5)


def test_two_body_rk4_reference(gs):
    """test_shooting.cpp:98-108: head-on pair under Euler T=1e4 vs an RK4 oracle."""
    q = np.array([[-1.0, 0, 0], [1.0, 0, 0]])
    p = np.array([[0.3, 0, 0], [-0.3, 0, 0]])
    cfg = ShootingConfig(sigma=1.0, timesteps=10000)
    fq, fp, _, _ = gs.shoot_forward(q, p, cfg, keep_trajectory=False)
    cfg4 = ShootingConfig(sigma=1.0, timesteps=2000, integrator=RK4)
    rq, rp, _, _ = gs.shoot_forward(q, p, cfg4, keep_trajectory=False)
    assert np.abs(fq - rq).max() < 1e-3 and np.abs(fp - rp).max() < 1e-3


def test_free_particle(gs):
    q = np.array([[0.5, -0.25, 2.0]])
    p = np.array([[1.0, 0.0, 0.0]])
    for t in (1, 7, 40):
        tr = gs.shoot_forward(q, p, ShootingConfig(sigma=3.0, timesteps=t))
        assert np.linalg.norm(tr.q[-1][0] - (q[0] + 2.0 * p[0])) < 1e-12
        assert np.array_equal(tr.p[-1], p)


@pytest.mark.parametrize("prec,tol", [(F64, F64_TOL), (F32, 1e-4)])
def test_evaluate_exact_matches_reference(gs, ref, prec, tol):
    n = 300
    q, p, t = uniform(n, 5.0, 461), sym_uniform(n, 0.3, 462), uniform(n, 5.0, 463)
    if prec == F32:
        q, p, t = f32(q), f32(p), f32(t)
    cfg = ShootingConfig(sigma=1.2, lambda_=0.7, timesteps=8, precision=prec)
    ev = gs.evaluate(q, p, t, cfg)
    rep, g, _, _ = ref.evaluate(q, p, t, 1.2, 0.7, 8, 0)
    assert ev.report["total"] == pytest.approx(rep[2], rel=tol)
    assert ev.report["energy"] == pytest.approx(rep[0], rel=tol)
    assert ev.report["residual_sse"] == pytest.approx(rep[3], rel=tol)
    assert rel_l2(ev.gradient, g) <= tol * 10


def test_backward_gradient_and_objective(gs, ref):
    n = 50
    q, p, t = uniform(n, 2.0, 441), sym_uniform(n, 0.3, 442), uniform(n, 2.0, 443)
    cfg = ShootingConfig(sigma=1.1, lambda_=0.8, timesteps=10)
    tr = gs.shoot_forward(q, p, cfg)
    g = gs.backward_gradient(tr, t, cfg)
    wq, wp = ref.shoot_forward(q, p, 1.1, 10)
    wg = ref.backward_gradient(wq, wp, t, 1.1, 0.8, 10)
    assert rel_l2(g, wg) <= F64_TOL
    obj = gs.objective(q, p, t, cfg)
    want = ref.objective(q, p, t, 1.1, 0.8, 10)
    assert obj["total"] == pytest.approx(want[2], rel=1e-12)


def test_gradient_zero_at_minimum(gs):
    q = uniform(4, 2.0, 431)
    cfg = ShootingConfig(sigma=1.0, timesteps=6)
    tr = gs.shoot_forward(q, np.zeros((4, 3)), cfg)
    assert not gs.backward_gradient(tr, q, cfg).any()


def test_warp_points_matches_reference(gs, ref):
    n = 200
    q, p = uniform(n, 1.5, 471), sym_uniform(n, 0.25, 472)
    cfg = ShootingConfig(sigma=0.8, timesteps=20)
    tr = gs.shoot_forward(q, p, cfg)
    x = uniform(97, 3.0, 473)
    y = gs.warp_points(tr, x, cfg)
    assert rel_l2(y, ref.warp_points(tr.q, tr.p, x, 0.8, 20)) <= 1e-12
    carried = gs.warp_points(tr, q, cfg)  # carrier points reproduce the endpoint
    assert np.abs(carried - tr.q[-1]).max() < 1e-10
    other = ShootingConfig(sigma=0.8, timesteps=21)
    with pytest.raises(ConfigMismatch):
        gs.warp_points(tr, q, other)
    with pytest.raises(ConfigMismatch):
        gs.backward_gradient(tr, q, other)


def test_nonfinite_reports_step(gs):
    q = np.array([[0.0, 0, 0], [0.1, 0, 0]])
    p = np.array([[1e200, 0, 0], [1e200, 0, 0]])
    with pytest.raises(NonFiniteState) as e:
        gs.shoot_forward(q, p, ShootingConfig(sigma=0.05, timesteps=4))
    assert 1 <= e.value.timestep <= 4


def test_config_errors(gs):
    with pytest.raises(ConfigError) as e:
        gs.shoot_forward(uniform(3, 1, 1), np.zeros((3, 3)),
                         ShootingConfig(sigma=-1, lambda_=0, timesteps=0, threshold_multiplier=0))
    assert e.value.violations == ["NonPositiveSigma", "NonPositiveLambda", "ZeroTimesteps",
                                  "NonPositiveThreshold"]


def test_empty_and_nonfinite_inputs(gs):
    with pytest.raises(ValueError):
        gs.hamiltonian(np.zeros((0, 3)), np.zeros((0, 3)), 1.0)
    with pytest.raises(ValueError):
        gs.hamiltonian(np.array([[np.nan, 0, 0]]), np.zeros((1, 3)), 1.0)


def test_bitwise_determinism(gs):
    q, p, t = uniform(400, 4.0, 481), sym_uniform(400, 0.3, 482), uniform(400, 4.0, 483)
    for prec in (F64, F32):
        cfg = ShootingConfig(sigma=1.0, timesteps=6, precision=prec)
        a = gs.evaluate(q, p, t, cfg)
        b = gs.evaluate(q, p, t, cfg)
        assert a.report["total"] == b.report["total"]
        assert np.array_equal(a.gradient, b.gradient)


# ---- Morton-ordered exact path with the FP32 underflow cutoff ------------------
def _flow_final(gs, q, p, cfg, steps):
    f = gs.flow(cfg, len(q))
    f.upload(q, p)
    f.advance(steps)
    f.sync()
    return f.download()


@pytest.mark.parametrize("n,sigma", [(4000, 0.01), (200_000, 0.0131)])
def test_exact_cutoff_is_bitwise_the_unskipped_sum(gs, n, sigma):
    """Skipping tiles beyond the FP32 underflow radius changes no bit: the
    same Morton-ordered sum without skipping gives identical states."""
    from paper_1907_04834_b200._lib import GS_FLAG_EXACT_MORTON
    rng = np.random.default_rng(n)
    q, p = rng.uniform(0, 1, (n, 3)), rng.normal(0, 1e-2, (n, 3))
    base = dict(sigma=sigma, timesteps=10, backend=EXACT, integrator=RK4, precision=F32)
    a = _flow_final(gs, q, p, ShootingConfig(exact_cutoff=True, **base), 2)
    b = _flow_final(gs, q, p, ShootingConfig(flags=GS_FLAG_EXACT_MORTON, **base), 2)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    c = _flow_final(gs, q, p, ShootingConfig(**base), 2)  # index-order sum: rounding only
    assert rel_l2(a[0], c[0]) < 1e-6 and rel_l2(a[1], c[1]) < 1e-5


def test_exact_cutoff_matches_reference(gs, port):
    n, sigma = 3000, 0.02
    q, p = f32(uniform(n, 1.0, 531)), f32(sym_uniform(n, 1e-3, 532))
    cfg = ShootingConfig(sigma=sigma, timesteps=4, backend=EXACT, integrator=RK4, precision=F32,
                         exact_cutoff=True)
    fq, fp, e, _ = gs.shoot_forward(q, p, cfg, keep_trajectory=False)
    w = port.shoot_forward(q, p, sigma, 4, integrator=1, keep_traj=False)
    assert rel_l2(fq, w["q"]) < F32_TRAJ_TOL and rel_l2(fp, w["p"]) < F32_TRAJ_TOL
    assert e == pytest.approx(w["energy"], rel=1e-5)


# ---- symmetric all-pairs (k_rhs_sym_f32x2: each unordered pair once) -----------
@pytest.fixture
def pairs(gs):
    def set_mode(mode):
        gs.set_exact_pairs(mode)
    yield set_mode
    gs.set_exact_pairs(-1)


# 512-point tiles below 35k points: one tile (diagonal only), 2 and 4 tiles
# (even T: the k = T/2 pairs taken once), 5 tiles (odd T), ragged last tiles
@pytest.mark.parametrize("n", [1, 2, 300, 513, 512 * 3 + 17, 512 * 4 + 5])
def test_symmetric_rhs_matches_reference(gs, ref, pairs, n):
    """Every unordered pair evaluated once and fed to both ends, as the
    reference's i < j sweep (kernel_exact.cpp:29-61): FP32 RHS to 1e-5 of the
    reference on the same FP32 inputs, to rounding of the gather kernel, and
    bitwise repeatable (the T partial slots are folded in fixed order)."""
    q, p = f32(uniform(n, 10.0, seed=n)), f32(sym_uniform(n, 1.0, seed=n + 1))
    pairs(2)
    h, dp, dq = gs.hamiltonian_with_gradients(q, p, 1.1, precision=F32)
    h2, dp2, dq2 = gs.hamiltonian_with_gradients(q, p, 1.1, precision=F32)
    assert np.array_equal(dp, dp2) and np.array_equal(dq, dq2) and h == h2
    wp, wq, wh = ref.exact_rhs(q, p, 1.1)
    assert rel_l2(dp, wp) < F32_RHS_TOL
    assert rel_l2(dq, wq) < F32_RHS_TOL
    assert abs(h - wh) <= F32_RHS_TOL * abs(wh)
    pairs(1)
    _, gp, gq = gs.hamiltonian_with_gradients(q, p, 1.1, precision=F32)
    assert rel_l2(dp, gp) < 2e-6 and rel_l2(dq, gq) < 2e-6


@pytest.mark.parametrize("n", [9_000, 40_000, 80_000])
def test_symmetric_tile_shapes_match_gather(gs, pairs, n):
    """The by-size tile shapes (512-point tiles from 8k, 768 from 35k, 1536 from
    75k points) against the gather kernel, to FP32 rounding."""
    rng = np.random.default_rng(n)
    q, p = rng.uniform(0, 1, (n, 3)), rng.normal(0, 1e-2, (n, 3))
    assert gs.exact_pairs_plan(n, F32) > 0
    _, dp, dq = gs.hamiltonian_with_gradients(q, p, 0.03, precision=F32)
    pairs(1)
    _, gp, gq = gs.hamiltonian_with_gradients(q, p, 0.03, precision=F32)
    assert rel_l2(dp, gp) < 2e-6 and rel_l2(dq, gq) < 2e-6


def test_symmetric_flow_matches_reference(gs, port, pairs):
    """RK4 flow through the symmetric kernel against the port's RK4 over the
    reference RHS (FP32 trajectory tolerance)."""
    n, sigma = 512 * 2 + 100, 0.05
    q, p = f32(uniform(n, 1.0, 541)), f32(sym_uniform(n, 1e-3, 542))
    pairs(2)
    cfg = ShootingConfig(sigma=sigma, timesteps=4, backend=EXACT, integrator=RK4, precision=F32)
    fq, fp, e, _ = gs.shoot_forward(q, p, cfg, keep_trajectory=False)
    w = port.shoot_forward(q, p, sigma, 4, integrator=1, keep_traj=False)
    assert rel_l2(fq, w["q"]) < F32_TRAJ_TOL and rel_l2(fp, w["p"]) < F32_TRAJ_TOL
    assert e == pytest.approx(w["energy"], rel=1e-5)


def test_exact_pairs_choice_is_validated(gs):
    with pytest.raises(ValueError):
        gs.set_exact_pairs(3)


# 512-point tiles below 40k points: one tile, 2 and 4 tiles (even T), 5 tiles
# (odd T), ragged
@pytest.mark.parametrize("n", [1, 300, 513, 512 * 3 + 11, 512 * 4 + 3])
def test_symmetric_hessian_products_match_reference(gs, ref, pairs, n):
    """k_hess_sym_f32x2: each unordered pair once, the j terms by symmetry
    (d -> -d, db -> -db), against the reference's hessian_products
    (kernel_exact.cpp:84-135) and the gather kernel; bitwise repeatable."""
    q, p = f32(uniform(n, 6.0, 95)), f32(sym_uniform(n, 1.0, 96))
    a, b = f32(sym_uniform(n, 1.0, 97)), f32(sym_uniform(n, 1.0, 98))
    pairs(2)
    got = gs.hessian_products(q, p, a, b, 1.2, precision=F32)
    again = gs.hessian_products(q, p, a, b, 1.2, precision=F32)
    want = ref.hessian_products(q, p, a, b, 1.2)
    pairs(1)
    gather = gs.hessian_products(q, p, a, b, 1.2, precision=F32)
    for g, g2, w, h in zip(got, again, want, gather):
        assert np.array_equal(g, g2)
        assert rel_l2(g, w) < 2e-5
        assert rel_l2(g, h) < 4e-6


def test_symmetric_evaluate_matches_reference(gs, ref, pairs):
    """evaluate() with the symmetric forward and adjoint kernels (FP32)."""
    n = 768 * 3 + 40
    q, p, t = f32(uniform(n, 9.0, 471)), f32(sym_uniform(n, 0.3, 472)), f32(uniform(n, 9.0, 473))
    pairs(2)
    cfg = ShootingConfig(sigma=1.2, lambda_=0.7, timesteps=6, precision=F32)
    ev = gs.evaluate(q, p, t, cfg)
    rep, g, _, _ = ref.evaluate(q, p, t, 1.2, 0.7, 6, 0)
    assert ev.report["total"] == pytest.approx(rep[2], rel=1e-4)
    assert rel_l2(ev.gradient, g) <= 1e-3


# FP64: 512-point tiles below 100k points (1024 above), diagonals in groups of
# 32 folded into a running sum; T = 1, 1, 2, 4 (even), 5 (odd)
@pytest.mark.parametrize("n", [1, 300, 513, 512 * 3 + 17, 512 * 4 + 5])
def test_symmetric_rhs_f64_matches_reference(gs, ref, pairs, n):
    q, p = uniform(n, 10.0, seed=n + 7), sym_uniform(n, 1.0, seed=n + 8)
    pairs(2)
    h, dp, dq = gs.hamiltonian_with_gradients(q, p, 1.1)
    h2, dp2, dq2 = gs.hamiltonian_with_gradients(q, p, 1.1)
    assert np.array_equal(dp, dp2) and np.array_equal(dq, dq2) and h == h2
    wp, wq, wh = ref.exact_rhs(q, p, 1.1)
    assert rel_l2(dp, wp) < 1e-13
    assert rel_l2(dq, wq) < 1e-12
    assert abs(h - wh) <= 1e-12 * abs(wh)


def test_symmetric_rhs_f64_groups_equal_gather(gs, pairs):
    """70k points: T = 137 tiles of 512, 69 diagonals in three groups (32 + 32 + 5): the
    symmetric FP64 sum against the gather kernel's to FP64 rounding."""
    n = 70_000
    rng = np.random.default_rng(70)
    q, p = rng.uniform(0, 1, (n, 3)), rng.normal(0, 1e-2, (n, 3))
    assert gs.exact_pairs_plan(n, F64) == 137
    _, dp, dq = gs.hamiltonian_with_gradients(q, p, 0.03)
    pairs(1)
    assert gs.exact_pairs_plan(n, F64) == 0
    _, gp, gq = gs.hamiltonian_with_gradients(q, p, 0.03)
    assert rel_l2(dp, gp) < 1e-13 and rel_l2(dq, gq) < 1e-12


_GROUPED = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1907_04834_b200 import F32, Geoshoot
gs = Geoshoot(0)
n = 100_000
rng = np.random.default_rng(100)
q, p = rng.uniform(0, 1, (n, 3)), rng.normal(0, 1e-2, (n, 3))
out, hp = [], []
a, b = rng.normal(0, 1, (n, 3)), rng.normal(0, 1, (n, 3))
for mode in (2, 2, 1):
    gs.set_exact_pairs(mode)
    out.append(gs.hamiltonian_with_gradients(q, p, 0.02, precision=F32)[1:])
    hp.append(np.concatenate(gs.hessian_products(q, p, a, b, 0.02, precision=F32)))
np.savez(sys.argv[2], a0=out[0][0], a1=out[0][1], b0=out[1][0], b1=out[1][1], g0=out[2][0], g1=out[2][1],
         h0=hp[0], h1=hp[1], hg=hp[2])
"""


@pytest.mark.parametrize("budget", ["1e6", ""])
def test_symmetric_grouped_diagonals(tmp_path, budget):
    """Problems whose tile slots exceed the partial budget (from ~1.5M points)
    run the symmetric kernel in diagonal groups of 32 folded into a running
    sum. GS_SYM_SLOT_BUDGET (read once per process, hence a subprocess) forces
    it at 100k points: 66 tiles, 34 diagonals in two groups, even T. Against
    the one-slot-per-tile run and the gather kernel: FP32 rounding; repeatable."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    if budget:
        env["GS_SYM_SLOT_BUDGET"] = budget
    f = tmp_path / f"g{budget or 'std'}.npz"
    subprocess.run([sys.executable, "-c", _GROUPED, root, str(f)], env=env, check=True, timeout=600)
    d = np.load(f)
    assert np.array_equal(d["a0"], d["b0"]) and np.array_equal(d["a1"], d["b1"])
    assert rel_l2(d["a0"], d["g0"]) < 2e-6 and rel_l2(d["a1"], d["g1"]) < 2e-6
    # Hessian products (768-point tiles: 131 tiles, 66 diagonals in 5 groups of 16)
    assert np.array_equal(d["h0"], d["h1"])
    assert rel_l2(d["h0"], d["hg"]) < 4e-6
    if budget:
        std = tmp_path / "std.npz"
        subprocess.run([sys.executable, "-c", _GROUPED, root, str(std)], check=True, timeout=600)
        s = np.load(std)
        assert not np.array_equal(d["a1"], s["a1"])  # a different (grouped) summation really ran
        assert not np.array_equal(d["h0"], s["h0"])
        assert rel_l2(d["h0"], s["h0"]) < 4e-6
        assert rel_l2(d["a0"], s["a0"]) < 2e-6 and rel_l2(d["a1"], s["a1"]) < 2e-6
