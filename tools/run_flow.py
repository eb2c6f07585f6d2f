"""Run a device-resident flow once (for ncu / compute-sanitizer captures).

  python tools/run_flow.py --backend bh --n 1000000 --steps 1 [--prec f32] [--rk4]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--backend", default="exact", choices=["exact", "bh"])
    ap.add_argument("--n", type=int, default=200000)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--prec", default="f32", choices=["f32", "f64"])
    ap.add_argument("--euler", action="store_true")
    ap.add_argument("--sigma", type=float, default=0.0131)
    ap.add_argument("--phases", action="store_true")
    ap.add_argument("--shape", default="cube", choices=["cube", "tube", "ellipsoid"])
    ap.add_argument("--amp", type=float, default=0.01)
    ap.add_argument("--no-profile", action="store_true", help="CUDA-graph replay (profiling forces eager launches)")
    a = ap.parse_args()
    import numpy as np
    from paper_1907_04834_b200 import BARNES_HUT, EULER, EXACT, F32, F64, RK4, Geoshoot, ShootingConfig
    rng = np.random.default_rng(2024)
    if a.shape == "cube":
        q, p = rng.uniform(0, 1, (a.n, 3)), rng.normal(0, 1e-2, (a.n, 3))
    else:
        from tests.util import ellipsoid, smooth_momenta, tube
        q = tube(a.n, seed=3) if a.shape == "tube" else ellipsoid(a.n, seed=44)
        p = smooth_momenta(q, a.amp, 4)
    gs = Geoshoot(0)
    cfg = ShootingConfig(sigma=a.sigma, timesteps=10, backend=BARNES_HUT if a.backend == "bh" else EXACT,
                         integrator=EULER if a.euler else RK4, precision=F32 if a.prec == "f32" else F64)
    f = gs.flow(cfg, a.n)
    f.upload(q, p)
    f.advance(a.warmup)
    f.sync()
    if not a.no_profile:
        f.profile(True)
    t0 = time.perf_counter()
    f.advance(a.steps)
    f.sync()
    dt = time.perf_counter() - t0
    pr = {} if a.no_profile else (f.profile_phases() if a.phases else f.profile_read())
    print(json.dumps({"backend": a.backend, "n": a.n, "steps": a.steps, "wall_s": dt,
                      "steps_per_s": a.steps / dt, "profile": pr}))


if __name__ == "__main__":
    main()
