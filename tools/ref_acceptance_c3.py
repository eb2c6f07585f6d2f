"""Acceptance criterion 3 (proj/tests/acceptance_main.cpp:166-220) computed
with the REFERENCE itself (oracle/_ref, compiled by path): the flat-rectangle
registration (N = 1202, sigma 2, lambda 1, T = 40, 60 L-BFGS iterations) with
the exact and the Barnes-Hut backends, and the relative residual gap the
criterion requires below 5 %. The reference's acceptance program cannot link
here (its Procrustes needs Eigen), so this restates criterion 3's computation
over the reference's own optimize(). Writes tests/golden/acceptance_c3_reference.json.

  python tools/ref_acceptance_c3.py      (~4 min, CPU)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import oracle
    R = oracle.ref()
    n = 1202
    flat = R.generate(1, n, 100.0, 4.0)
    bent = R.generate(2, n, 100.0, 4.0, 0.5235987755982988)
    out = {}
    for backend, name in ((0, "exact"), (1, "bh")):
        t0 = time.time()
        r = R.optimize(flat, bent, 2.0, 1.0, 40, backend=backend, max_iterations=60)
        out[name] = {"reason": r["reason"], "iterations": r["iterations"],
                     "residual": float(r["trace"][-1][3]), "cpu_s": time.time() - t0}
    out["gap"] = abs(out["bh"]["residual"] - out["exact"]["residual"]) / out["exact"]["residual"]
    out["criterion3_pass"] = out["gap"] < 0.05
    with open(os.path.join(ROOT, "tests", "golden", "acceptance_c3_reference.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
