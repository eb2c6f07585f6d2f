"""BASELINE config 2 (N = 20k ellipsoid, sigma 3, 20 Euler steps) through
shoot_forward: wall time with graphs, then the per-phase event times
(gs_profile: kernel / build / build phases; graphs off while profiling).

  python tools/profile_c2.py [--prec f32|f64] [--backend bh|exact]
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
    ap.add_argument("--prec", default="f32")
    ap.add_argument("--backend", default="bh")
    ap.add_argument("--n", type=int, default=20000)
    a = ap.parse_args()
    from paper_1907_04834_b200 import BARNES_HUT, EXACT, F32, F64, Geoshoot, ShootingConfig
    from tests.util import ellipsoid, smooth_momenta
    gs = Geoshoot(0)
    q = ellipsoid(a.n, seed=44)
    p = smooth_momenta(q, 0.5, 43)
    cfg = ShootingConfig(sigma=3.0, timesteps=20, backend=BARNES_HUT if a.backend == "bh" else EXACT,
                         precision=F32 if a.prec == "f32" else F64)
    run = lambda: gs.shoot_forward(q, p, cfg, keep_trajectory=False)  # noqa: E731
    run()
    best = 1e30
    for _ in range(5):
        t0 = time.perf_counter()
        run()
        best = min(best, time.perf_counter() - t0)
    gs.profile(True)
    run()
    ph = gs.profile_phases()
    gs.profile(False)
    out = {"wall_ms": best * 1e3}
    out.update({k: round(v["ms"] / 20, 4) for k, v in ph.items() if v["count"]})
    out["counts"] = {k: v["count"] for k, v in ph.items()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
