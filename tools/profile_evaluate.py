"""One config-3 `evaluate` (N = 50k tube, sigma = 5, T = 20, FP32) for kernel
launch lists: python tools/profile_evaluate.py [--backend bh|exact] [--reps R]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--backend", default="bh", choices=["bh", "exact"])
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--n", type=int, default=50000)
    ap.add_argument("--flow", action="store_true")
    a = ap.parse_args()
    import numpy as np
    from paper_1907_04834_b200 import BARNES_HUT, EXACT, F32, Geoshoot, ShootingConfig
    from tests.util import smooth_momenta, tube
    gs = Geoshoot(0)
    q = tube(a.n, seed=3)
    tgt, _, _, _ = gs.shoot_forward(q, smooth_momenta(q, 0.01, 4), ShootingConfig(sigma=5.0, timesteps=20),
                                    keep_trajectory=False)
    cfg = ShootingConfig(sigma=5.0, lambda_=100.0, timesteps=20,
                         backend=BARNES_HUT if a.backend == "bh" else EXACT, precision=F32)
    p0 = np.zeros_like(q) + 1e-3
    if a.flow:  # the same forward as a device-resident flow, per-phase GPU times
        f = gs.flow(cfg, a.n)
        f.upload(q, p0)
        f.advance(1)
        f.sync()
        f.upload(q, p0)
        f.profile(True)
        f.advance(20)
        f.sync()
        print(json.dumps({"flow_phases": f.profile_phases()}), flush=True)
        return
    for r in range(a.reps):
        t0 = time.perf_counter()
        ev = gs.evaluate(q, p0, tgt, cfg)
        print(json.dumps({"rep": r, "s": time.perf_counter() - t0, "stats": ev.stats}), flush=True)


if __name__ == "__main__":
    main()
