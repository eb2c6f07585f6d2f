"""Composition of one graph-replayed flow step on the device (gs_trace):
every traced kernel's start time (%globaltimer), grouped per step, and each
kernel's share = time from its start to the next traced kernel's start (its
run time plus the launch gap after it). Host-side events cannot time inside a
captured graph; this can.

  python tools/trace_step.py [--config c2|c4bh|c4bh0] [--prec f32|f64] [--backend bh|exact]

c4bh: config 4 (N = 1M, RK4) through shoot_forward (10 steps; the flow
diverges from step 4); c4bh0: its first steps only (no divergence).
"""
import argparse
import collections
import json
import os
import re
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
UNITS = {1: "tree.cu", 2: "bh.cu", 3: "epilogue.cu"}


def kernel_names():
    """(unit, line) -> name of the __global__ function enclosing that line."""
    out = {}
    for u, f in UNITS.items():
        text = open(os.path.join(ROOT, "paper_1907_04834_b200", "csrc", f)).read()
        starts = []  # (line of the kernel's name, name)
        for m in re.finditer(r"__global__", text):
            k = re.compile(r"\b(k_\w+)\s*\(").search(text, m.end())
            if k:
                starts.append((text.count("\n", 0, k.start()) + 1, k.group(1)))
        nlines = text.count("\n") + 1
        j, cur = 0, "?"
        for i in range(1, nlines + 1):
            while j < len(starts) and starts[j][0] <= i:
                cur = starts[j][1]
                j += 1
            out[(u, i)] = cur
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--prec", default="f32")
    ap.add_argument("--backend", default="bh")
    a = ap.parse_args()
    from paper_1907_04834_b200 import BARNES_HUT, EXACT, F32, F64, RK4, Geoshoot, ShootingConfig
    from tests.util import ellipsoid, smooth_momenta
    gs = Geoshoot(0)
    prec = F32 if a.prec == "f32" else F64
    backend = BARNES_HUT if a.backend == "bh" else EXACT
    if a.config == "c2":
        q = ellipsoid(20000, seed=44)
        p = smooth_momenta(q, 0.5, 43)
        cfg = ShootingConfig(sigma=3.0, timesteps=20, backend=backend, precision=prec)
    else:
        from bench import workload
        q, p = workload(1_000_000)
        cfg = ShootingConfig(sigma=0.0131, timesteps=10, backend=backend, integrator=RK4, precision=prec)
    if a.config == "c4bh0":
        # config 4's first RK4 steps only (its flow diverges from step 4 on:
        # extent 1e9, most points in runs of equal 63-bit keys)
        f = gs.flow(cfg, len(q))
        f.upload(q, p)
        f.advance(3)
        f.sync()
        f.upload(q, p)
        gs.trace(True)
        f.advance(3)  # graph-replayed from step 1 (captured above): steps 1-2 measured
        f.sync()
    else:
        run = lambda: gs.shoot_forward(q, p, cfg, keep_trajectory=False)  # noqa: E731
        run()
        gs.trace(True)
        run()
    tr = gs.trace_read()
    gs.trace(False)
    names = kernel_names()
    ev = [(names.get((u, l), f"{u}:{l}"), t) for u, l, t in tr]
    # a step ends with its final stage's epilogue (which also advances the
    # step counter); skip the first two steps (eager, capture)
    stages = 4 if a.config.startswith("c4") else 1
    steps, cur, epis = [], [], 0
    for nm, t in ev:
        cur.append((nm, t))
        if nm == "k_fwd_epi":
            epis += 1
            if epis % stages == 0:
                steps.append(cur)
                cur = []
    share = collections.defaultdict(list)
    step_ns = []
    for k in range(0 if a.config == "c4bh0" else 2, len(steps)):
        st = steps[k]
        nxt = steps[k + 1][0][1] if k + 1 < len(steps) else None
        if nxt is None:
            continue
        step_ns.append(nxt - st[0][1])
        per = collections.defaultdict(float)
        for i, (nm, t) in enumerate(st):
            t2 = st[i + 1][1] if i + 1 < len(st) else nxt
            per[nm] += t2 - t
        for nm, v in per.items():
            share[nm].append(v)
    out = {"config": a.config, "prec": a.prec, "backend": a.backend, "steps_traced": len(step_ns),
           "step_us": float(np.mean(step_ns)) / 1e3 if step_ns else None,
           "kernels_per_step": len(steps[-1]) if steps else None,
           "share_us": {nm: round(float(np.mean(v)) / 1e3, 2) for nm, v in
                        sorted(share.items(), key=lambda x: -np.mean(x[1]))}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
