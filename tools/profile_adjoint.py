"""One config-3 exact evaluate() (N = 50k tube, sigma 5, T = 20, FP32): the
adjoint's Hessian-product kernel (k_hess_f32x2) for ncu.

  ncu --set full -k regex:k_hess_f32x2 -c 1 python tools/profile_adjoint.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1907_04834_b200 import EXACT, F32, Geoshoot, ShootingConfig
    from tests.util import smooth_momenta, tube
    gs = Geoshoot(0)
    q = tube(50000, seed=3)
    tgt, _, _, _ = gs.shoot_forward(q, smooth_momenta(q, 0.01, 4), ShootingConfig(sigma=5.0, timesteps=20),
                                    keep_trajectory=False)
    cfg = ShootingConfig(sigma=5.0, lambda_=100.0, timesteps=int(sys.argv[1]) if len(sys.argv) > 1 else 2,
                         backend=EXACT, precision=F32)
    ev = gs.evaluate(q, np.full_like(q, 1e-3), tgt, cfg)
    print(ev.report)


if __name__ == "__main__":
    main()
