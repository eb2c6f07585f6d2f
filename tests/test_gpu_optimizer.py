"""Registration optimizer: L-BFGS + strong Wolfe over
p0 (optimizer.cpp:215-351) driving the device evaluate(), against the
reference's own optimize() on the same problem. With FP64 evaluations that
agree to ~1e-13, the search takes the same steps: same termination reason and
iteration count, trace and optimum within 1e-6 relative."""
import numpy as np
import pytest

from paper_1907_04834_b200 import BARNES_HUT, EXACT, F32, F64, ShootingConfig
from tests.util import rel_l2

pytestmark = pytest.mark.gpu


def problem(ref, n=100):
    q = ref.generate(1, n, 60.0, 4.0)           # flat rectangle (synthetic.cpp)
    t = ref.generate(2, n, 60.0, 4.0, 0.5)      # bent rectangle, 0.5 rad
    return q, t


@pytest.mark.parametrize("backend", [EXACT, BARNES_HUT])
def test_optimize_matches_reference(gs, ref, backend):
    q, t = problem(ref)
    cfg = ShootingConfig(sigma=4.0, lambda_=1.0, timesteps=8, backend=backend, precision=F64)
    got = gs.optimize(q, t, cfg, max_iterations=15)
    want = ref.optimize(q, t, 4.0, 1.0, 8, backend=backend, max_iterations=15)
    assert got["reason"] == want["reason"]
    assert got["iterations"] == want["iterations"]
    assert len(got["trace"]) == len(want["trace"])
    np.testing.assert_allclose(got["trace"][:, 1:5], want["trace"][:, 1:5], rtol=1e-6, atol=1e-12)
    assert rel_l2(got["p0"], want["p0"]) <= 1e-6
    # it registers: the objective decreases monotonically
    assert (np.diff(got["trace"][:, 1]) < 0).all()


def test_optimize_f32_reaches_reference_objective(gs, ref):
    q, t = problem(ref)
    cfg = ShootingConfig(sigma=4.0, lambda_=1.0, timesteps=8, precision=F32)
    got = gs.optimize(q, t, cfg, max_iterations=15)
    want = ref.optimize(q, t, 4.0, 1.0, 8, max_iterations=15)
    assert got["trace"][-1, 1] == pytest.approx(want["trace"][-1, 1], rel=1e-3)


def test_identity_problem_stops_at_start(gs):
    q = np.random.default_rng(1).uniform(0, 2, (20, 3))
    out = gs.optimize(q, q, ShootingConfig(sigma=1.0, timesteps=4), max_iterations=5)
    assert out["reason"] == "gradient_tolerance" and out["iterations"] == 0
    assert not out["p0"].any()


def test_optimize_batch_equals_single(gs, ref):
    """Config-5 batching: concurrent subjects give the single-subject results."""
    subj = []
    for k in range(3):
        q = ref.generate(1, 80 + 10 * k, 60.0, 4.0)
        t = ref.generate(2, 80 + 10 * k, 60.0, 4.0, 0.3 + 0.1 * k)
        subj.append((q, t))
    cfg = ShootingConfig(sigma=4.0, lambda_=1.0, timesteps=6, backend=BARNES_HUT, precision=F32)
    out = gs.optimize_batch([q for q, _ in subj], [t for _, t in subj], cfg, max_iterations=8)
    for k, (q, t) in enumerate(subj):
        one = gs.optimize(q, t, cfg, max_iterations=8)
        assert np.array_equal(out["p0"][k], one["p0"])  # bitwise: deterministic kernels
        assert out["iterations"][k] == one["iterations"]


def test_register_subjects_single_rank(gs, ref):
    """shard.register_subjects (config 5 across GPUs) on one rank: the rank's
    block is every subject, results equal optimize_batch's."""
    from paper_1907_04834_b200.shard import register_subjects
    qs = [ref.generate(3, 60 + 5 * k, 60.0, 4.0) for k in range(3)]
    ts = [ref.generate(4, 60 + 5 * k, 60.0, 4.0, 0.2) for k in range(3)]
    cfg = ShootingConfig(sigma=4.0, lambda_=1.0, timesteps=4, backend=BARNES_HUT, precision=F32)
    res = register_subjects(gs, qs, ts, cfg, max_iterations=4)
    out = gs.optimize_batch(qs, ts, cfg, max_iterations=4)
    assert [r["subject"] for r in res] == [0, 1, 2]
    for k, r in enumerate(res):
        assert np.array_equal(r["p0"], out["p0"][k])
        assert r["iterations"] == out["iterations"][k]


def test_evaluate_batch_equals_single(gs):
    """gs_evaluate_batch: subjects of different N on concurrent streams give the
    one-at-a-time results bitwise; evaluate_subjects (one rank) the same."""
    from paper_1907_04834_b200.shard import evaluate_subjects
    from tests.util import ellipsoid, smooth_momenta
    qs = [ellipsoid(400 + 150 * k, seed=70 + k) for k in range(3)]
    ps = [smooth_momenta(q, 0.01, 80 + k) for k, q in enumerate(qs)]
    ts = [q + 0.3 for q in qs]
    for backend in (EXACT, BARNES_HUT):
        cfg = ShootingConfig(sigma=3.0, lambda_=10.0, timesteps=5, backend=backend, precision=F32)
        evs = gs.evaluate_batch(qs, ps, ts, cfg)
        for q, p, t, e in zip(qs, ps, ts, evs):
            one = gs.evaluate(q, p, t, cfg)
            assert np.array_equal(e.gradient, one.gradient)
            assert e.report == one.report
        res = evaluate_subjects(gs, qs, ps, ts, cfg)
        assert [r["subject"] for r in res] == [0, 1, 2]
        assert all(np.array_equal(r["gradient"], e.gradient) for r, e in zip(res, evs))
