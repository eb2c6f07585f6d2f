import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_1907_04834_b200 import Geoshoot, F32
gs = Geoshoot(0)
rng = np.random.default_rng(1)
for n, far in ((1_000_000, 1e3), (1_000_000, 1e5), (4_000_000, 1e3)):
    q = np.concatenate([rng.uniform(0, 1, (n, 3)), [[-far] * 3, [far] * 3]])
    p = np.zeros_like(q)
    t = gs.build_tree(q, p, precision=F32)
    d = t.download()
    s = np.sort(d["key_hi"]); eq = s[1:] == s[:-1]
    # run lengths
    starts = np.flatnonzero(np.concatenate([[True], ~eq]))
    lens = np.diff(np.concatenate([starts, [len(s)]]))
    for r in range(2): gs.build_tree(q, p, precision=F32)
    gs.sync() if hasattr(gs, "sync") else None
    t0 = time.perf_counter()
    for r in range(5): t = gs.build_tree(q, p, precision=F32)
    t.node_count()
    print(n, far, "tie pairs", int(eq.sum()), "max run", int(lens.max()), "runs>32", int((lens > 32).sum()),
          "build ms", (time.perf_counter() - t0) / 5 * 1e3)
