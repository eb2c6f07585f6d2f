import sys
sys.path.insert(0, '.')
from bench import workload
from paper_1907_04834_b200 import Geoshoot, F32, BARNES_HUT, RK4, ShootingConfig
gs = Geoshoot(0)
n = 1_000_000
q, p = workload(n)
cfg = ShootingConfig(sigma=0.0131, timesteps=10, backend=BARNES_HUT, integrator=RK4, precision=F32)
f = gs.flow(cfg, n)
f.upload(q, p)
f.advance(5); f.sync()
qf, pf = f.download()
for r in range(3):
    t = gs.build_tree(qf, pf, precision=F32)
print(t.node_count())
