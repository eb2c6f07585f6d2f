"""Octree build timing at config 4 (N = 1M unit cube, FP32): per-phase CUDA-event
times of the builds inside a Barnes-Hut RK4 flow (gs_flow_profile_phases).

  python tools/profile_build.py [--n N] [--steps K]
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv python tools/profile_build.py --steps 1   # per kernel

Algorithmic bytes per point: bench.py BUILD_BYTES_PER_POINT.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    a = ap.parse_args()
    from paper_1907_04834_b200 import BARNES_HUT, F32, RK4, Geoshoot, ShootingConfig
    from bench import BUILD_BYTES_PER_POINT, workload
    gs = Geoshoot(0)
    q, p = workload(a.n)
    # config 4 at 1M; at other n the momenta scale by 1M / n so the velocity
    # field (a sum over the sigma-ball) stays config 4's -- the unscaled flow
    # diverges at 4M (positions fly off, the root box dwarfs the cloud)
    sigma = 0.0131
    p = p * (1e6 / a.n)
    cfg = ShootingConfig(sigma=sigma, timesteps=10, backend=BARNES_HUT, integrator=RK4,
                         precision=F32)
    f = gs.flow(cfg, a.n)
    f.upload(q, p)
    f.advance(a.warmup)
    f.sync()
    f.upload(q, p)
    f.profile(True)
    f.advance(a.steps)
    f.sync()
    ph = f.profile_phases(6)
    qf, _ = f.download()
    finite = bool(np.isfinite(qf).all())
    builds = max(1, ph["build"]["count"])
    out = {k: v["ms"] / max(1, v["count"]) for k, v in ph.items()}
    out["n"] = a.n
    out["builds"] = builds
    out["finite"] = finite
    out["build_gbs_algorithmic"] = BUILD_BYTES_PER_POINT * a.n / (out["build"] * 1e-3) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
