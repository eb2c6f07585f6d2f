"""Symmetric vs gather exact FP32 RHS (gs_set_exact_pairs 2 vs 1): agreement
with each other and with the FP64 RHS, and the time of one flow step.

  python tools/check_sym.py [--n 200000 1000000] [--time-n 1000000]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel(a, b):
    import numpy as np
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="*", default=[3000, 20000, 200000])
    ap.add_argument("--time-n", type=int, default=1000000)
    ap.add_argument("--time-steps", type=int, default=1)
    ap.add_argument("--modes", type=int, nargs="*", default=[1, 2, 1, 2])
    ap.add_argument("--f64", action="store_true")
    a = ap.parse_args()
    import numpy as np
    from paper_1907_04834_b200 import EXACT, F32, F64, RK4, Geoshoot, ShootingConfig
    gs = Geoshoot(0)
    for n in a.n:
        rng = np.random.default_rng(7 + n)
        q, p = rng.uniform(0, 1, (n, 3)), rng.normal(0, 1e-2, (n, 3))
        sigma = 0.0131 * (1e6 / n) ** (1 / 3)
        out = {}
        for mode in (1, 2):
            gs.set_exact_pairs(mode)
            h, dp, dq = gs.hamiltonian_with_gradients(q, p, sigma, precision=F32)
            h2, dp2, dq2 = gs.hamiltonian_with_gradients(q, p, sigma, precision=F32)
            out[mode] = (h, dp, dq, bool(np.array_equal(dp, dp2) and np.array_equal(dq, dq2)))
        gs.set_exact_pairs(-1)
        r = {"n": n, "sigma": sigma,
             "sym_vs_gather_dp": rel(out[2][1], out[1][1]), "sym_vs_gather_dq": rel(out[2][2], out[1][2]),
             "repeatable": [out[1][3], out[2][3]], "h": [out[1][0], out[2][0]]}
        if n <= 200000:
            h64, dp64, dq64 = gs.hamiltonian_with_gradients(q, p, sigma, precision=F64)
            r.update(gather_vs_f64=[rel(out[1][1], dp64), rel(out[1][2], dq64)],
                     sym_vs_f64=[rel(out[2][1], dp64), rel(out[2][2], dq64)], h64=h64)
        print(json.dumps(r), flush=True)
    if a.time_n:
        n = a.time_n
        rng = np.random.default_rng(2024)
        q, p = rng.uniform(0, 1, (n, 3)), rng.normal(0, 1e-4, (n, 3))
        for mode in a.modes:
            gs.set_exact_pairs(mode)
            cfg = ShootingConfig(sigma=0.0131, timesteps=10, backend=EXACT, integrator=RK4,
                                 precision=F64 if a.f64 else F32)
            f = gs.flow(cfg, n)
            f.upload(q, p)
            f.advance(1)
            f.sync()
            t0 = time.perf_counter()
            f.advance(a.time_steps)
            f.sync()
            dt = (time.perf_counter() - t0) / a.time_steps
            qq, pp = f.download()
            print(json.dumps({"mode": mode, "n": n, "s_per_rk4_step": dt,
                              "pairs_per_s": 4.0 * n * n / dt, "q_sum": float(qq.sum())}), flush=True)
            del f
        gs.set_exact_pairs(-1)




def hess_main():
    """python tools/check_sym.py hess N: exact evaluate() (forward + adjoint), gather vs symmetric."""
    import numpy as np
    from paper_1907_04834_b200 import EXACT, F32, Geoshoot, ShootingConfig
    from tests.util import smooth_momenta, tube
    n = int(sys.argv[2])
    gs = Geoshoot(0)
    q = tube(n, seed=5)
    p = smooth_momenta(q, 1.0, 6)
    t = q + 0.5
    cfg = ShootingConfig(sigma=5.0, lambda_=100.0, timesteps=20, backend=EXACT, precision=F32)
    for mode in (1, 2, 1, 2):
        gs.set_exact_pairs(mode)
        gs.evaluate(q, p, t, cfg)
        t0 = time.perf_counter()
        ev = gs.evaluate(q, p, t, cfg)
        dt = time.perf_counter() - t0
        print(json.dumps({"mode": mode, "n": n, "evaluate_s": dt, "total": ev.report["total"],
                          "grad_norm": float(np.linalg.norm(ev.gradient))}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "hess":
        hess_main()
    else:
        main()
