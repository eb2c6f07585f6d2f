"""Time the exact dense warp (gs_warp_points, FP32): M eval points advected
through a T-step trajectory of N points. python tools/time_warp.py [N] [M]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    from paper_1907_04834_b200 import EXACT, F32, Geoshoot, ShootingConfig
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 200000
    rng = np.random.default_rng(5)
    q, p = rng.uniform(0, 1, (n, 3)), rng.normal(0, 1e-3, (n, 3))
    x = rng.uniform(0, 1, (m, 3))
    gs = Geoshoot(0)
    cfg = ShootingConfig(sigma=0.0131, timesteps=4, backend=EXACT, precision=F32)
    traj = gs.shoot_forward(q, p, cfg, keep_trajectory=True)
    gs.warp_points(traj, x, cfg)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        gs.warp_points(traj, x, cfg)
        best = min(best, time.perf_counter() - t0)
    print(json.dumps({"n": n, "m": m, "steps": 4, "best_s": best,
                      "gpair_per_s": 4.0 * n * m / best / 1e9}))


if __name__ == "__main__":
    main()
