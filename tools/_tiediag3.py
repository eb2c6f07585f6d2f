import sys, numpy as np
sys.path.insert(0, '.')
from paper_1907_04834_b200 import Geoshoot, F32
gs = Geoshoot(0)
rng = np.random.default_rng(1)
for n, far in ((1_000_000, 1e7), (100_000, 1e7)):
    q = np.concatenate([rng.uniform(0, 1, (n, 3)), [[-far] * 3, [far] * 3]])
    t = gs.build_tree(q, np.zeros_like(q), precision=F32)
    print(n, t.node_count())
