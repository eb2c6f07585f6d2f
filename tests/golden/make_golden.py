"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the container that holds /root/reference (it needs oracle/_ref, the
reference's own hot-path sources compiled by path, see oracle/Makefile):

    make -C oracle all && python tests/golden/make_golden.py

Every fixture records its inputs (seeded, synthetic: BASELINE.json names no
public data set) and the reference outputs. RK4 has no reference
implementation (shooting.hpp:16-18); its fixture is produced by the oracle
port's RK4 composed over the reference RHS and says so in `provenance`.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from tests.util import ellipsoid, f32, smooth_momenta, sphere, sym_uniform, uniform  # noqa: E402


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)
    print("wrote", name, {k: getattr(v, "shape", v) for k, v in arrays.items()})


def main():
    R = oracle.ref()
    P = oracle.port()

    # kernel_exact known answers (test_kernel_exact.cpp style, N=3 and N=64)
    for n in (3, 64):
        q, p = uniform(n, 4.0, 21 + n), sym_uniform(n, 1.0, 22 + n)
        a, b = sym_uniform(n, 1.0, 23 + n), sym_uniform(n, 1.0, 24 + n)
        dp, dq, h = R.exact_rhs(q, p, 1.7)
        hp = R.hessian_products(q, p, a, b, 1.7)
        x = uniform(7, 4.0, 25 + n)
        save(f"exact_n{n}", provenance="reference", q=q, p=p, alpha=a, beta=b, sigma=1.7,
             H=h, H_direct=R.hamiltonian(q, p, 1.7), dH_dp=dp, dH_dq=dq, pq=hp[0], pp=hp[1],
             qq=hp[2], qp=hp[3], x=x, v=R.exact_velocity(x, q, p, 1.7))

    # BASELINE config 1: N=1024 unit sphere, N(0, 0.01^2) momenta, sigma 0.2, 10 Euler steps
    q, p = sphere(1024, 7), np.random.default_rng(8).normal(0, 0.01, (1024, 3))
    tq, tp = R.shoot_forward(q, p, 0.2, 10)
    q32, p32 = f32(q), f32(p)
    tq32, tp32 = R.shoot_forward(q32, p32, 0.2, 10)
    save("config1", provenance="reference", q0=q, p0=p, sigma=0.2, timesteps=10,
         q_T=tq[-1], p_T=tp[-1], energy=R.hamiltonian(q, p, 0.2), H_T=R.hamiltonian(tq[-1], tp[-1], 0.2),
         q0_f32=q32, p0_f32=p32, q_T_f32in=tq32[-1], p_T_f32in=tp32[-1])

    # octree: keys / leaf order / node count (integer work, bit-exact)
    for name, (q, p) in {
        "cube": (uniform(2000, 1.0, 1), sym_uniform(2000, 1.0, 2)),
        "duplicates": (np.concatenate([np.full((10, 3), 0.5), uniform(190, 2.0, 6)]),
                       sym_uniform(200, 1.0, 7)),
    }.items():
        t = R.tree(q, p)
        d = t.dump()
        kh, kl = P.morton_keys(q)
        # reference DFS leaf order (children 0..7; bucket members ascending)
        order, stack = [], [0]
        while stack:
            k = stack.pop()
            if d["leaf"][k]:
                run, i = [], d["first_point"][k]
                while i >= 0:
                    run.append(i)
                    i = d["next_point"][i]
                order.extend(sorted(run))
            else:
                stack.extend(c for c in d["children"][k][::-1] if c >= 0)
        save(f"tree_{name}", provenance="reference tree + port midpoint-replay keys", q=q, p=p,
             node_count=t.node_count(), order=np.array(order, np.int32), key_hi=kh, key_lo=kl,
             count=d["count"], actual_min=d["actual_min"], actual_max=d["actual_max"])

    # Barnes-Hut RHS at 3 sigma (config-2-like ellipsoid, smaller N)
    q = ellipsoid(2000, seed=44)
    p = smooth_momenta(q, 0.5, 43)
    dp, dq, per = R.tree(q, p).bh_rhs(3.0, 9.0, threads=8)
    save("bh_ellipsoid", provenance="reference", q=q, p=p, sigma=3.0, threshold=9.0, dH_dp=dp,
         dH_dq=dq, per_query=per)

    # evaluate (fused forward + adjoint), exact and BH
    n = 300
    q = np.stack([np.linspace(0, 60, n), np.random.default_rng(81).uniform(-2, 2, n), np.zeros(n)], 1)
    p, t = sym_uniform(n, 0.05, 82), q + np.array([0.0, 0.5, 0.1])
    for backend in (0, 1):
        rep, g, stats, _ = R.evaluate(q, p, t, 2.0, 1.0, 10, backend, threads=8)
        save(f"evaluate_{'bh' if backend else 'exact'}", provenance="reference", q0=q, p0=p, target=t,
             sigma=2.0, lam=1.0, timesteps=10, report=rep, gradient=g, stats=stats)

    # RK4 (no reference implementation): port RK4 composed over the reference RHS
    q = uniform(500, 1.0, 31)
    p = np.random.default_rng(32).normal(0, 1e-2, (500, 3))
    w = P.shoot_forward(q, p, 0.05, 10, integrator=1, keep_traj=False)
    save("rk4_exact", provenance="oracle port RK4 over the reference RHS (no reference RK4)",
         q0=q, p0=p, sigma=0.05, timesteps=10, q_T=w["q"], p_T=w["p"], energy=w["energy"])


if __name__ == "__main__":
    main()
