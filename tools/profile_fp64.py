"""Exact FP64 right-hand sides at config 4's distribution (for ncu).

  ncu --set full -k regex:k_rhs_f64 -c 1 python tools/profile_fp64.py [N]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1907_04834_b200 import F64, Geoshoot
    from bench import SIGMA, workload
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
    q, p = workload(n)
    gs = Geoshoot(0)
    gs.hamiltonian_with_gradients(q, p, SIGMA, precision=F64)
    print("done", n)


if __name__ == "__main__":
    main()
