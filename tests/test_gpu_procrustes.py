"""Rigid pre-alignment (procrustes.cpp:7-58). The
reference needs Eigen (absent here), so it cannot be built: parity is pinned
to the reference's own test scenarios (test_pipeline.cpp:68-135: identity,
exact recovery of a known rigid transform, noisy data beats doing nothing,
degenerate input refused) and to a numpy Kabsch restatement (test-only)."""
import numpy as np
import pytest

from paper_1907_04834_b200 import DegenerateConfiguration

pytestmark = pytest.mark.gpu


def rot(ax, ay, az):
    cx, sx, cy, sy, cz, sz = np.cos(ax), np.sin(ax), np.cos(ay), np.sin(ay), np.cos(az), np.sin(az)
    Rx = np.array([[1, 0, 0], [0, cx, -sx], [0, sx, cx]])
    Ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
    Rz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1]])
    return Rz @ Ry @ Rx


def kabsch(s, t):
    sm, tm = s.mean(0), t.mean(0)
    H = (s - sm).T @ (t - tm)
    U, S, Vt = np.linalg.svd(H)
    d = np.sign(np.linalg.det(Vt.T @ U.T))
    R = Vt.T @ np.diag([1, 1, d]) @ U.T
    return R, tm - R @ sm


def test_identity(gs):
    q = np.random.default_rng(1).uniform(-1, 1, (50, 3))
    R, t, y = gs.procrustes_align(q, q)
    assert np.abs(R - np.eye(3)).max() < 1e-12 and np.abs(t).max() < 1e-12
    assert np.abs(y - q).max() < 1e-12


def test_exact_recovery(gs):
    rng = np.random.default_rng(2)
    s = rng.uniform(-5, 5, (200, 3))
    R0 = rot(0.3, -1.1, 2.0)
    t0 = np.array([4.0, -2.5, 7.25])
    tgt = s @ R0.T + t0
    R, t, y = gs.procrustes_align(s, tgt)
    assert np.abs(R - R0).max() < 1e-12 and np.abs(t - t0).max() < 1e-11
    assert np.abs(y - tgt).max() < 1e-11
    assert np.linalg.det(R) == pytest.approx(1.0, abs=1e-12)


def test_matches_kabsch_and_reduces_residual(gs):
    rng = np.random.default_rng(3)
    s = rng.normal(0, 3, (5000, 3))
    tgt = s @ rot(1.0, 0.2, -0.7).T + np.array([1, 2, 3]) + rng.normal(0, 0.3, s.shape)
    R, t, y = gs.procrustes_align(s, tgt)
    Rk, tk = kabsch(s, tgt)
    assert np.abs(R - Rk).max() < 1e-12 and np.abs(t - tk).max() < 1e-10
    assert np.linalg.norm(y - tgt) < np.linalg.norm(s - tgt)


def test_reflection_is_corrected(gs):
    rng = np.random.default_rng(4)
    s = rng.normal(0, 1, (100, 3))
    tgt = s * np.array([1, 1, -1])  # a mirror image: best proper rotation, det +1
    R, _, _ = gs.procrustes_align(s, tgt)
    assert np.linalg.det(R) == pytest.approx(1.0, abs=1e-12)


def test_degenerate(gs):
    with pytest.raises(DegenerateConfiguration):
        gs.procrustes_align(np.zeros((2, 3)), np.zeros((2, 3)))
    line = np.outer(np.linspace(0, 1, 20), [1.0, 2.0, 3.0])
    with pytest.raises(DegenerateConfiguration):
        gs.procrustes_align(line, line + 1.0)
