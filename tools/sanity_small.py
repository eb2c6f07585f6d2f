"""Small end-to-end exercise of every device path (a smoke run of all kernels):
exact (index order, Morton cutoff), BH walks (independent, group, windows,
literal-mean-dot, shards by index), evaluate (forward + adjoint), warp,
Procrustes, batched subjects."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_04834_b200 import BARNES_HUT, EXACT, F32, F64, RK4, Geoshoot, ShootingConfig  # noqa: E402

gs = Geoshoot(0)
rng = np.random.default_rng(1)
n = 3000
q, p = rng.uniform(0, 1, (n, 3)), rng.normal(0, 1e-2, (n, 3))
t = q + 0.01
for prec in (F32, F64):
    for backend in (EXACT, BARNES_HUT):
        for lmd in (False, True):
            cfg = ShootingConfig(sigma=0.05, timesteps=3, backend=backend, precision=prec,
                                 integrator=RK4, literal_mean_dot=lmd,
                                 exact_cutoff=(prec == F32 and backend == EXACT and lmd))
            gs.shoot_forward(q, p, cfg, keep_trajectory=False)
            cfg_e = ShootingConfig(sigma=0.05, timesteps=3, backend=backend, precision=prec,
                                   literal_mean_dot=lmd)  # the adjoint is Euler's
            gs.evaluate(q, p, t, cfg_e)
            tr = gs.shoot_forward(q, p, cfg_e)
            gs.warp_points(tr, q[:100] + 0.001, cfg_e)
            f = gs.flow(cfg, n)
            f.upload(q, p)
            f.set_shard(0, n // 2)
            for s in range(4):
                f.stage(s)
            f.sync()
tree = gs.build_tree(q, p, precision=F32)
tree.bh_hamiltonian_gradients(0.05, 0.15)
gs.procrustes_align(q, q @ np.array([[0, -1, 0], [1, 0, 0], [0, 0, 1.0]]).T + 0.5)
cfg = ShootingConfig(sigma=0.05, timesteps=3, backend=BARNES_HUT, precision=F32)
gs.evaluate_batch([q, q[:1000]], [p, p[:1000]], [t, t[:1000]], cfg)
print("sanity ok")
