"""Config 3 (50k tube, sigma 5, lambda 100, T = 20): FP32 evaluate() gradients
of the gather and the symmetric exact kernels against the FP64 evaluate(),
and the L-BFGS runs (100 iterations) of both FP32 formulations.

  python tools/c3_gradient_accuracy.py [--optimize]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tests.util import smooth_momenta, tube  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--optimize", action="store_true")
    a = ap.parse_args()
    from paper_1907_04834_b200 import EXACT, F32, F64, Geoshoot, ShootingConfig
    gs = Geoshoot(0)
    q = tube(50000, seed=3)
    tgt, _, _, _ = gs.shoot_forward(q, smooth_momenta(q, 0.01, 4), ShootingConfig(sigma=5.0, timesteps=20),
                                    keep_trajectory=False)
    rng = np.random.default_rng(9)
    for amp in (1e-3, 5e-3):
        p0 = amp * rng.standard_normal(q.shape)
        c64 = ShootingConfig(sigma=5.0, lambda_=100.0, timesteps=20, backend=EXACT, precision=F64)
        ref = gs.evaluate(q, p0, tgt, c64)
        out = {"p0_amplitude": amp, "total_f64": ref.report["total"]}
        for mode, name in ((1, "gather"), (2, "symmetric")):
            gs.set_exact_pairs(mode)
            ev = gs.evaluate(q, p0, tgt, ShootingConfig(sigma=5.0, lambda_=100.0, timesteps=20,
                                                       backend=EXACT, precision=F32))
            g = ev.gradient
            out[name] = {"total_rel_err": abs(ev.report["total"] - ref.report["total"]) / abs(ref.report["total"]),
                         "gradient_rel_l2": float(np.linalg.norm(g - ref.gradient) / np.linalg.norm(ref.gradient))}
        gs.set_exact_pairs(-1)
        print(json.dumps(out), flush=True)
    if a.optimize:
        for mode, name in ((1, "gather"), (2, "symmetric")):
            gs.set_exact_pairs(mode)
            cfg = ShootingConfig(sigma=5.0, lambda_=100.0, timesteps=20, backend=EXACT, precision=F32)
            t0 = time.perf_counter()
            r = gs.optimize(q, tgt, cfg, max_iterations=100)
            dt = time.perf_counter() - t0
            print(json.dumps({"optimize": name, "s": dt, "iterations": r["iterations"],
                              "evaluations": r["evaluations"], "reason": r["reason"],
                              "last_trace_row": [float(x) for x in r["trace"][-1]] if len(r["trace"]) else None,
                              "s_per_evaluation": dt / max(1, r["evaluations"])}), flush=True)
        gs.set_exact_pairs(-1)


if __name__ == "__main__":
    main()
