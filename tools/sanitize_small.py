"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): octree builds (FP32 and FP64, a clustered set with depth-32
buckets and chunk-spanning nodes), every Barnes-Hut query kind through every
walk, a graph-replayed RK4 flow, exact and Barnes-Hut evaluate(), and a
two-shard multi-device context.

  compute-sanitizer --tool memcheck python tools/sanitize_small.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1907_04834_b200 import (BARNES_HUT, EXACT, F32, F64, RK4, Geoshoot,
                                       ShootingConfig)
    from tests.util import ellipsoid, smooth_momenta, sym_uniform, uniform
    gs = Geoshoot(0)
    rng = np.random.default_rng(1)
    sets = {
        "cube": (uniform(3000, 1.0, 1), sym_uniform(3000, 0.01, 2), 0.05),
        "ellipsoid": (ellipsoid(2500, seed=3), None, 3.0),
        "cluster": (np.concatenate([uniform(1500, 1e-7, 8), uniform(500, 1.0, 9)]),
                    sym_uniform(2000, 1.0, 10), 0.1),
    }
    for name, (q, p, sigma) in sets.items():
        if p is None:
            p = smooth_momenta(q, 0.5, 4)
        for prec in (F64, F32):
            t = gs.build_tree(q, p, precision=prec)
            t.download()
            for kernel, windows in ((0, 0), (1, 1), (3, 7), (4, 32)):
                gs.set_bh_walk(kernel, windows)
                t.bh_hamiltonian_gradients(sigma, 3 * sigma)
                t.query_stats()
                a, b = sym_uniform(len(q), 1.0, 11), sym_uniform(len(q), 1.0, 12)
                t.accumulate_adjoints(a, b)
                t.bh_hessian_products(a, b, sigma, 3 * sigma)
                x = rng.uniform(q.min(0), q.max(0), (100, 3))
                t.bh_velocity(x, sigma, 3 * sigma)
                t.bh_point_gradients(x, sym_uniform(100, 0.1, 13), sigma, 3 * sigma)
            gs.set_bh_walk(-1, -1)
    q, p = uniform(4000, 1.0, 21), np.random.default_rng(22).normal(0, 1e-2, (4000, 3))
    for backend in (EXACT, BARNES_HUT):
        cfg = ShootingConfig(sigma=0.05, timesteps=4, backend=backend, integrator=RK4, precision=F32)
        f = gs.flow(cfg, len(q))
        f.upload(q, p)
        f.advance(3)  # graph capture + replay after the first step
        f.sync()
        f.download()
        cfg2 = ShootingConfig(sigma=0.05, lambda_=1.0, timesteps=4, backend=backend, precision=F64)
        gs.evaluate(q, p, q + 0.01, cfg2)
    m = Geoshoot(devices=[0, 0])
    for backend in (EXACT, BARNES_HUT):
        cfg = ShootingConfig(sigma=0.05, lambda_=1.0, timesteps=3, backend=backend, precision=F32)
        m.shoot_forward(q, p, cfg, keep_trajectory=False)
        m.evaluate(q, p, q + 0.01, cfg)
    m.close()
    gs.close()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
