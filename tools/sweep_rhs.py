"""Tuning sweep of the FP32 all-pairs RHS kernel variants (GS_RHS_VARIANT).

Each variant runs in its own process (the variant is latched once per
process): an exact FP32 RK4 flow at N points, kernel time from CUDA events on
the flow's stream. Prints one JSON line per variant.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(n, steps):
    sys.path.insert(0, ROOT)
    import numpy as np
    from paper_1907_04834_b200 import EXACT, F32, RK4, Geoshoot, ShootingConfig
    rng = np.random.default_rng(1)
    q, p = rng.uniform(0, 1, (n, 3)), rng.normal(0, 1e-2, (n, 3))
    gs = Geoshoot(0)
    f = gs.flow(ShootingConfig(sigma=0.0131, timesteps=10, backend=EXACT, integrator=RK4,
                               precision=F32), n)
    f.upload(q, p)
    f.advance(1)
    f.sync()
    f.profile(True)
    f.advance(steps)
    f.sync()
    pr = f.profile_read()
    ms = pr["kernel_ms"] / pr["kernel_launches"]
    print(json.dumps({"variant": int(os.environ.get("GS_RHS_VARIANT", "0")), "n": n,
                      "kernel_ms": ms, "gpair_per_s": n * float(n) / ms / 1e6}), flush=True)


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
    if os.environ.get("GS_SWEEP_CHILD"):
        one(n, 2)
    else:
        vs = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else range(4)
        for v in vs:
            env = dict(os.environ, GS_RHS_VARIANT=str(v), GS_SWEEP_CHILD="1")
            subprocess.run([sys.executable, __file__, str(n)], env=env, check=False)
