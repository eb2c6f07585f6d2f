"""CPU checks of the checker itself (no GPU): the oracle port (oracle/port.c)
is pinned against the reference's own outputs -- the committed golden
fixtures (tests/golden/, generated from oracle/_ref by make_golden.py) and,
where the by-path reference build is present, the reference run live -- plus
the reference's own known-answer tests restated (test_kernel_exact.cpp,
test_octree.cpp, test_shooting.cpp)."""
import glob
import os

import numpy as np
import pytest

from tests.util import rel_l2, sym_uniform, uniform

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def test_golden_fixtures_present():
    names = {os.path.basename(f)[:-4] for f in glob.glob(os.path.join(GOLD, "*.npz"))}
    assert {"exact_n3", "exact_n64", "config1", "tree_cube", "tree_duplicates", "bh_ellipsoid",
            "evaluate_exact", "evaluate_bh", "rk4_exact"} <= names


# ---- port vs the reference's golden outputs ---------------------------------
@pytest.mark.parametrize("n", [3, 64])
def test_port_exact_matches_golden(port, n):
    g = gold(f"exact_n{n}")
    dp, dq, h = port.exact_rhs(g["q"], g["p"], float(g["sigma"]))
    assert np.array_equal(dp, g["dH_dp"]) and np.array_equal(dq, g["dH_dq"]) and h == g["H"]
    assert port.hamiltonian(g["q"], g["p"], float(g["sigma"])) == g["H_direct"]
    hp = port.hessian_products(g["q"], g["p"], g["alpha"], g["beta"], float(g["sigma"]))
    for got, key in zip(hp, ("pq", "pp", "qq", "qp")):
        assert np.array_equal(got, g[key])
    assert np.array_equal(port.exact_velocity(g["x"], g["q"], g["p"], float(g["sigma"])), g["v"])


def test_port_config1_matches_golden(port):
    g = gold("config1")
    w = port.shoot_forward(g["q0"], g["p0"], 0.2, 10, keep_traj=False)
    assert np.array_equal(w["q"], g["q_T"]) and np.array_equal(w["p"], g["p_T"])
    assert w["energy"] == pytest.approx(float(g["energy"]), rel=1e-13)
    w = port.shoot_forward(g["q0_f32"], g["p0_f32"], 0.2, 10, keep_traj=False)
    assert np.array_equal(w["q"], g["q_T_f32in"])


@pytest.mark.parametrize("name", ["cube", "duplicates"])
def test_port_tree_matches_golden(port, name):
    g = gold(f"tree_{name}")
    t = port.tree(g["q"], g["p"])
    assert t.node_count() == int(g["node_count"])
    assert np.array_equal(t.leaf_order(), g["order"])
    kh, kl = port.morton_keys(g["q"])
    assert np.array_equal(kh, g["key_hi"]) and np.array_equal(kl, g["key_lo"])
    # Morton order (stable by (key_hi, key_lo), then index) == reference DFS leaf order
    order = np.lexsort((np.arange(len(kh)), kl, kh))
    assert np.array_equal(order, g["order"])
    d = t.dump()
    assert np.array_equal(d["count"], g["count"])
    assert np.array_equal(d["actual_min"], g["actual_min"])


def test_port_bh_matches_golden(port):
    g = gold("bh_ellipsoid")
    dp, dq, per = port.tree(g["q"], g["p"]).bh_rhs(float(g["sigma"]), float(g["threshold"]))
    assert np.array_equal(dp, g["dH_dp"]) and np.array_equal(dq, g["dH_dq"])
    assert np.array_equal(per, g["per_query"])


@pytest.mark.parametrize("kind", ["exact", "bh"])
def test_port_evaluate_matches_golden(port, kind):
    g = gold(f"evaluate_{kind}")
    rep, grad = port.evaluate(g["q0"], g["p0"], g["target"], float(g["sigma"]), float(g["lam"]),
                              int(g["timesteps"]), backend=1 if kind == "bh" else 0)
    assert np.array_equal(rep, g["report"]) and np.array_equal(grad, g["gradient"])


def test_port_rk4_matches_golden(port):
    g = gold("rk4_exact")
    w = port.shoot_forward(g["q0"], g["p0"], 0.05, 10, integrator=1, keep_traj=False)
    assert np.array_equal(w["q"], g["q_T"]) and np.array_equal(w["p"], g["p_T"])


# ---- port vs the reference, live (when oracle/_ref is built) -----------------
def test_port_bit_exact_vs_reference_live(port, ref):
    n = 300
    q, p = uniform(n, 8.0, 1), sym_uniform(n, 1.0, 2)
    a, b = sym_uniform(n, 1.0, 3), sym_uniform(n, 1.0, 4)
    x, y = ref.exact_rhs(q, p, 1.1), port.exact_rhs(q, p, 1.1)
    assert all(np.array_equal(u, v) for u, v in zip(x, y))
    rt, pt = ref.tree(q, p), port.tree(q, p)
    rd, pd = rt.dump(), pt.dump()
    assert all(np.array_equal(rd[k], pd[k]) for k in rd)
    rt.accumulate(a, b)
    pt.accumulate(a, b)
    assert all(np.array_equal(u, v) for u, v in
               zip(rt.bh_hessprod(a, b, 1.1, 3.3), pt.bh_hessprod(a, b, 1.1, 3.3)))
    tq, tp = ref.shoot_forward(q, p * 0.1, 1.1, 5, backend=1)
    w = port.shoot_forward(q, p * 0.1, 1.1, 5, backend=1)
    assert np.array_equal(tq, w["traj_q"]) and np.array_equal(tp, w["traj_p"])
    wq = ref.warp_points(tq, tp, q[:40] + 0.3, 1.1, 5, backend=1)
    assert np.array_equal(wq, port.warp(tq, tp, q[:40] + 0.3, 1.1, backend=1))


# ---- reference known-answer tests, restated on the oracle ----------------------
def test_kat_kernel_exact(port):
    # single point: H = |p|^2 (G(0) = 1); dH/dp = 2p, dH/dq = 0 (test_kernel_exact.cpp:65-69,136-142)
    q, p = np.array([[1.0, 2.0, 3.0]]), np.array([[0.5, -1.0, 0.25]])
    dp, dq, h = port.exact_rhs(q, p, 3.0)
    assert np.array_equal(dp, 2 * p) and not dq.any() and h == 1.3125
    # G(6; sigma = 2) = e^-4.5 : one unit momentum at distance 6
    q2 = np.array([[0.0, 0, 0], [6.0, 0, 0]])
    v = port.exact_velocity(q2[:1], q2[1:], np.array([[1.0, 0, 0]]), 2.0)
    assert v[0, 0] == pytest.approx(np.exp(-4.5), rel=1e-15)


def test_kat_fd_gradients(port):
    # central differences, h = 1e-5 (test_kernel_exact.cpp:143-164)
    q, p = uniform(5, 2.0, 51), sym_uniform(5, 1.0, 52)
    dp, dq, _ = port.exact_rhs(q, p, 1.3)
    h = 1e-5
    for i in range(5):
        for a in range(3):
            e = np.zeros_like(q)
            e[i, a] = h
            fq = (port.hamiltonian(q + e, p, 1.3) - port.hamiltonian(q - e, p, 1.3)) / (2 * h)
            fp = (port.hamiltonian(q, p + e, 1.3) - port.hamiltonian(q, p - e, 1.3)) / (2 * h)
            assert abs(dq[i, a] - fq) <= 1e-6 * max(abs(fq), abs(dq[i, a]), 1e-8)
            assert abs(dp[i, a] - fp) <= 1e-6 * max(abs(fp), abs(dp[i, a]), 1e-8)


def test_kat_octree(port):
    corners = np.array([[1.0 if i & 1 else -1.0, 1.0 if i & 2 else -1.0, 1.0 if i & 4 else -1.0]
                        for i in range(8)])
    t = port.tree(corners, np.zeros((8, 3)))
    assert t.node_count() == 9  # test_octree.cpp:91-110
    dup = np.concatenate([np.full((10, 3), 0.5), [[2.0, 2.0, 2.0]]])
    t = port.tree(dup, sym_uniform(11, 1.0, 66))
    d = t.dump()
    assert t.node_count() <= 2 * (32 + 2)  # bucket at the depth cap (test_octree.cpp:270-296)
    assert max(d["count"][d["leaf"]]) == 10


def test_rk4_two_body_convergence(port):
    # Euler (T = 1e4) vs RK4 (T = 2e3) on the head-on pair, test_shooting.cpp:98-108
    q = np.array([[-1.0, 0, 0], [1.0, 0, 0]])
    p = np.array([[0.3, 0, 0], [-0.3, 0, 0]])
    e = port.shoot_forward(q, p, 1.0, 10000, keep_traj=False)
    r = port.shoot_forward(q, p, 1.0, 2000, integrator=1, keep_traj=False)
    assert np.abs(e["q"] - r["q"]).max() < 1e-3 and np.abs(e["p"] - r["p"]).max() < 1e-3


def test_fd_adjoint(port):
    # the discrete adjoint matches finite differences of the objective (test_shooting.cpp:174-200)
    n = 3
    q, p, t = uniform(n, 2.0, 441), sym_uniform(n, 0.3, 442), uniform(n, 2.0, 443)
    _, g = port.evaluate(q, p, t, 1.1, 0.8, 10)
    h = 1e-5
    for i in range(n):
        for a in range(3):
            e = np.zeros_like(p)
            e[i, a] = h
            fp = (port.evaluate(q, p + e, t, 1.1, 0.8, 10)[0][2] -
                  port.evaluate(q, p - e, t, 1.1, 0.8, 10)[0][2]) / (2 * h)
            assert abs(g[i, a] - fp) <= 1e-5 * max(abs(fp), abs(g[i, a]), 1e-6)
    assert rel_l2(g, g) == 0.0


def test_ref_literal_mean_dot_build():
    """The GEOSHOOT_BH_LITERAL_MEAN_DOT build of the reference (oracle/Makefile)
    changes only the aggregate dot (dH/dq), never dH/dp or the exact path."""
    import oracle
    if not os.path.exists(oracle.REF_LMD_SO):
        pytest.skip("literal-mean-dot reference build absent")
    rng = np.random.default_rng(17)
    q, p = rng.uniform(0, 1, (800, 3)), rng.uniform(-1, 1, (800, 3))
    R, L = oracle.ref(), oracle.ref_lmd()
    dp0, dq0, per0 = R.tree(q, p).bh_rhs(0.03, 0.09)
    dp1, dq1, per1 = L.tree(q, p).bh_rhs(0.03, 0.09)
    assert np.array_equal(per0, per1) and np.array_equal(dp0, dp1)
    assert not np.array_equal(dq0, dq1)
    a = R.exact_rhs(q, p, 0.03)
    b = L.exact_rhs(q, p, 0.03)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
