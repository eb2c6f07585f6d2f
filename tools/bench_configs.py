"""Time every BASELINE.json configuration on the B200 path (and, where the
reference can finish in seconds, the reference CPU path on the same box).

  python tools/bench_configs.py [--cpu] > profiles/r01_configs.jsonl

Configs (BASELINE.json "configs", seeded synthetic stand-ins):
  C1  exact FP64, N=1024 unit sphere, sigma 0.2, 10 Euler steps
  C2  BH (3 sigma gate), N=20k ellipsoid (30,15,10) + N(0,0.5^2) jitter,
      smooth momenta amplitude 0.5, sigma 3, 20 Euler steps, FP64 + FP32 (+ exact)
  C3  evaluate (forward + adjoint), N=50k tube, sigma 5, lambda 100, 20 steps,
      FP32, exact and BH -- one evaluation (the optimizer's unit of work)
  C4  see bench.py (N=1M, RK4)
  C5  8 independent subjects x N=30k ellipsoids (per-GPU share of 64), BH,
      sigma 3, 20 steps, FP32 -- one evaluation each
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tests.util import ellipsoid, smooth_momenta, sphere, tube  # noqa: E402


def timed(fn, reps=3):
    fn()
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cpu", action="store_true", help="also time the reference CPU path")
    ap.add_argument("--full", action="store_true", help="also run full C3 / C5 registrations")
    a = ap.parse_args()
    from paper_1907_04834_b200 import BARNES_HUT, EXACT, F32, F64, Geoshoot, ShootingConfig
    gs = Geoshoot(0)
    ref = None
    if a.cpu:
        import oracle
        ref = oracle.ref() if oracle.have_ref() else None
    threads = os.cpu_count() or 1

    # C1
    q = sphere(1024, 7)
    p = np.random.default_rng(8).normal(0, 0.01, (1024, 3))
    cfg = ShootingConfig(sigma=0.2, timesteps=10, backend=EXACT, precision=F64)
    t = timed(lambda: gs.shoot_forward(q, p, cfg, keep_trajectory=False))
    rec = {"config": "C1", "what": "shoot_forward exact FP64 N=1024 T=10 Euler", "gpu_s": t,
           "pairs_per_s": 10 * 1024 ** 2 / t}
    if ref:
        rec["cpu_s"] = timed(lambda: ref.shoot_forward(q, p, 0.2, 10), reps=1)
        rec["cpu_threads"] = 1
    print(json.dumps(rec), flush=True)

    # C2
    q = ellipsoid(20000, seed=44)
    p = smooth_momenta(q, 0.5, 43)
    for prec, name in ((F64, "FP64"), (F32, "FP32")):
        for backend, bname in ((BARNES_HUT, "BH"), (EXACT, "exact")):
            cfg = ShootingConfig(sigma=3.0, timesteps=20, backend=backend, precision=prec)
            try:
                t = timed(lambda: gs.shoot_forward(q, p, cfg, keep_trajectory=False))
                status = "ok"
            except Exception as e:  # divergent flow still timed up to the error
                t, status = float("nan"), type(e).__name__
            _, _, _, st = (gs.shoot_forward(q, p, cfg, keep_trajectory=False) if status == "ok"
                           else (None, None, None, {}))
            print(json.dumps({"config": "C2", "what": f"shoot_forward {bname} {name} N=20k T=20",
                              "gpu_s": t, "status": status,
                              "interactions": (st.get("direct_interactions", 0) +
                                               st.get("approximated_interactions", 0))}), flush=True)
    if ref:
        t = timed(lambda: ref.shoot_forward(q, p, 3.0, 20, backend=1), reps=1)
        print(json.dumps({"config": "C2", "what": "reference shoot_forward BH FP64 N=20k T=20",
                          "cpu_s": t, "cpu_threads": threads}), flush=True)

    # C3: one evaluation; target from a smooth ground-truth field at a
    # well-conditioned amplitude (amp 1.0 diverges)
    q = tube(50000, seed=3)
    p_true = smooth_momenta(q, 0.01, 4)
    tgt, _, _, _ = gs.shoot_forward(q, p_true, ShootingConfig(sigma=5.0, timesteps=20),
                                    keep_trajectory=False)
    p0 = np.zeros_like(q)
    for backend, bname in ((EXACT, "exact"), (BARNES_HUT, "BH")):
        cfg = ShootingConfig(sigma=5.0, lambda_=100.0, timesteps=20, backend=backend, precision=F32)
        t = timed(lambda: gs.evaluate(q, p0 + 1e-3, tgt, cfg), reps=2)
        ev = gs.evaluate(q, p0 + 1e-3, tgt, cfg)
        print(json.dumps({"config": "C3", "what": f"evaluate {bname} FP32 N=50k T=20", "gpu_s": t,
                          "stats": ev.stats}), flush=True)

    # C5: 8 subjects (one GPU's share of 64), one BH evaluation each
    rng = np.random.default_rng(5)
    subj = []
    for k in range(8):
        ax = (rng.uniform(25, 35), rng.uniform(12, 18), rng.uniform(8, 12))
        qk = ellipsoid(30000, axes=ax, jitter=0.0, seed=100 + k)
        pk = smooth_momenta(qk, 0.008, 200 + k)
        cfg = ShootingConfig(sigma=3.0, lambda_=1.0, timesteps=20, backend=BARNES_HUT, precision=F32)
        tk, _, _, _ = gs.shoot_forward(qk, pk, cfg, keep_trajectory=False)
        subj.append((qk, tk, cfg))
    t0 = time.perf_counter()
    for qk, tk, cfg in subj:
        gs.evaluate(qk, np.zeros_like(qk) + 1e-3, tk, cfg)
    t = time.perf_counter() - t0
    print(json.dumps({"config": "C5", "what": "8 subjects x evaluate BH FP32 N=30k T=20 (sequential)",
                      "gpu_s": t, "per_subject_s": t / 8}), flush=True)
    cfg5 = subj[0][2]
    qs, ts = [q for q, _, _ in subj], [t for _, t, _ in subj]
    ps = [np.zeros_like(q) + 1e-3 for q in qs]
    gs.evaluate_batch(qs, ps, ts, cfg5)  # warm the per-subject contexts
    t0 = time.perf_counter()
    gs.evaluate_batch(qs, ps, ts, cfg5)
    t = time.perf_counter() - t0
    print(json.dumps({"config": "C5", "what": "8 subjects x evaluate BH FP32 N=30k T=20 "
                      "(gs_evaluate_batch: concurrent streams)", "gpu_s": t, "per_subject_s": t / 8}),
          flush=True)

    if a.full:
        # full registrations (BASELINE configs 3 and 5: L-BFGS)
        q = tube(50000, seed=3)
        tgt, _, _, _ = gs.shoot_forward(q, smooth_momenta(q, 0.01, 4), ShootingConfig(sigma=5.0, timesteps=20),
                                        keep_trajectory=False)
        for backend, bname in ((EXACT, "exact"), (BARNES_HUT, "BH")):
            cfg = ShootingConfig(sigma=5.0, lambda_=100.0, timesteps=20, backend=backend, precision=F32)
            t0 = time.perf_counter()
            out = gs.optimize(q, tgt, cfg, max_iterations=100)
            t = time.perf_counter() - t0
            print(json.dumps({"config": "C3", "what": f"optimize {bname} FP32 N=50k T=20, 100 iterations",
                              "gpu_s": t, "iterations": out["iterations"],
                              "evaluations": out["evaluations"], "reason": out["reason"]}), flush=True)
        t0 = time.perf_counter()
        res = gs.optimize_batch(qs, ts, cfg5, max_iterations=50)
        t = time.perf_counter() - t0
        print(json.dumps({"config": "C5", "what": "8 subjects x optimize BH FP32 N=30k T=20, 50 iterations "
                          "(gs_optimize_batch, one GPU's share of 64)", "gpu_s": t,
                          "iterations": res["iterations"], "evaluations": res["evaluations"]}),
              flush=True)


if __name__ == "__main__":
    main()
