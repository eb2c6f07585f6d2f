"""One BASELINE config-3 evaluate (N = 50k tube, sigma 5, T = 20, FP32) through
the Barnes-Hut path, for kernel launch lists of the dense-regime walks.

  ncu --metrics gpu__time_duration.sum --csv python tools/profile_dense.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1907_04834_b200 import BARNES_HUT, F32, Geoshoot, ShootingConfig
    from tests.util import smooth_momenta, tube
    gs = Geoshoot(0)
    q = tube(50000, seed=3)
    tgt, _, _, _ = gs.shoot_forward(q, smooth_momenta(q, 0.01, 4), ShootingConfig(sigma=5.0, timesteps=20),
                                    keep_trajectory=False)
    p = np.full_like(q, 1e-3)
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    cfg = ShootingConfig(sigma=5.0, lambda_=100.0, timesteps=steps, backend=BARNES_HUT, precision=F32)
    gs.evaluate(q, p, tgt, cfg)
    t0 = time.perf_counter()
    ev = gs.evaluate(q, p, tgt, cfg)
    print("evaluate_s", time.perf_counter() - t0, ev.stats)


if __name__ == "__main__":
    main()
