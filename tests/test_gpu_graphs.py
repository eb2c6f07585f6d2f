"""CUDA-graph replay of integrator steps (capi.cu flow_advance) is bit-identical
to eager stepping: the same launches with the same arguments, only replayed.
Eager mode is forced with GS_GRAPHS=0 in a child process (the switch is read
once per process)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np
from paper_1907_04834_b200 import Geoshoot, ShootingConfig, EXACT, BARNES_HUT, F32, F64, EULER, RK4
from tests.util import uniform, sym_uniform
out = {}
gs = Geoshoot()
q, p, t = uniform(700, 3.0, 11), sym_uniform(700, 0.2, 12), uniform(700, 3.0, 13)
for be in (EXACT, BARNES_HUT):
    for prec in (F64, F32):
        for integ in (EULER, RK4):
            cfg = ShootingConfig(sigma=0.4, timesteps=7, backend=be, precision=prec, integrator=integ)
            fq, fp, e, st = gs.shoot_forward(q, p, cfg, keep_trajectory=False)
            # a second call with the same configuration replays the step graph
            # left by the first from step 1 on (graphs on; eager otherwise)
            fq2, fp2, _, _ = gs.shoot_forward(q, p, cfg, keep_trajectory=False)
            assert np.array_equal(fq, fq2) and np.array_equal(fp, fp2)
            key = f"{be}_{prec}_{integ}"
            out[key + "_q"], out[key + "_p"] = fq, fp
            out[key + "_e"] = np.array([e])
            out[key + "_direct"] = np.array([st["direct_interactions"]])
            f = gs.flow(cfg, len(q))
            f.upload(q, p)
            f.advance(3)
            f.advance(2)
            out[key + "_fq"], out[key + "_fp"] = f.download()
np.savez(sys.argv[1], **out)
"""


def _run(tmp_path, graphs):
    path = str(tmp_path / f"g{graphs}.npz")
    env = dict(os.environ, GS_GRAPHS=str(graphs))
    subprocess.run([sys.executable, "-c", CHILD, path], check=True, cwd=ROOT, env=env, timeout=600)
    return np.load(path)


def test_graph_replay_bitwise_equals_eager(tmp_path):
    g, e = _run(tmp_path, 1), _run(tmp_path, 0)
    assert sorted(g.files) == sorted(e.files)
    for k in g.files:
        assert np.array_equal(g[k], e[k]), k



LIFETIME = r"""
import numpy as np
from paper_1907_04834_b200 import Geoshoot, ShootingConfig, BARNES_HUT
g = Geoshoot(0)
q = np.random.default_rng(1).uniform(0, 1, (2000, 3))
p = np.zeros_like(q)
f = g.flow(ShootingConfig(sigma=0.05, timesteps=2, backend=BARNES_HUT), len(q))
f.upload(q, p)
f.advance(1)
t = g.build_tree(q, p)
g.close()      # the context goes first ...
del f, t       # ... its flow and tree are still destroyable (gs_destroy detaches them)
print("ok")
"""


def test_flow_and_tree_outlive_their_context():
    """gs_destroy before gs_flow_destroy / gs_tree_free (e.g. objects kept
    alive by a traceback past a fixture's teardown) must not touch the dead
    context."""
    r = subprocess.run([sys.executable, "-c", LIFETIME], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), (r.returncode, r.stderr[-2000:])


def test_kernel_trace_inside_graph(gs):
    """gs_trace: the device-side start times of the build, walk and epilogue
    kernels of graph-replayed Barnes-Hut steps (tools/trace_step.py)."""
    from paper_1907_04834_b200 import BARNES_HUT, F32, ShootingConfig
    from tests.util import sym_uniform, uniform
    q, p = uniform(3000, 1.0, 31), sym_uniform(3000, 0.01, 32)
    cfg = ShootingConfig(sigma=0.05, timesteps=4, backend=BARNES_HUT, precision=F32)
    gs.shoot_forward(q, p, cfg, keep_trajectory=False)
    gs.trace(True)
    try:
        gs.shoot_forward(q, p, cfg, keep_trajectory=False)
        tr = gs.trace_read()
    finally:
        gs.trace(False)
    units = {u for u, _, _ in tr}
    assert units == {1, 2, 3}  # tree.cu, bh.cu, epilogue.cu
    t = np.array([v for _, _, v in tr], np.float64)
    assert len(tr) >= 4 * 15 and (np.diff(t) >= 0).all()  # 4 steps in stream order
    with pytest.raises(ValueError):
        gs.trace_read()  # tracing off
