"""Target sharding on real kernels (the per-stage path of a multi-GPU run,
SURVEY.md §8e), emulated with two flows on one GPU: each owns half of the
targets, runs its stages, and the updated halves are exchanged between the
two record buffers after every stage exactly as the in-place all-gather of
shard.ShardedFlow would. Exact: the result must be bit-identical to one
unsharded flow (a shard launches under the full problem's plan, so its
per-target sums are the same); Barnes-Hut: equal to FP32 summation-order
rounding (same interaction sets).
A Barnes-Hut shard walks only its own targets, taken by index from records
put in Morton order at set_shard (so a shard is a compact region).
"""
import numpy as np
import pytest
import torch

from paper_1907_04834_b200 import BARNES_HUT, EXACT, F32, RK4, ShootingConfig
from paper_1907_04834_b200.shard import records_view
from tests.util import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture
def gather(gs):
    # shards run the gather kernel (k_rhs_f32x2): compare against the same
    # formulation on one flow (the unsharded default at this size is the
    # symmetric kernel, equal to FP32 rounding -- checked below)
    gs.set_exact_pairs(1)
    yield
    gs.set_exact_pairs(-1)


@pytest.mark.parametrize("backend", [EXACT, BARNES_HUT])
def test_two_shards_equal_one_flow(gs, gather, backend):
    n = 60_000
    rng = np.random.default_rng(77)
    q, p = rng.uniform(0, 1, (n, 3)), rng.normal(0, 1e-2, (n, 3))
    cfg = ShootingConfig(sigma=0.03, timesteps=10, backend=backend, integrator=RK4, precision=F32)
    one = gs.flow(cfg, n)
    one.upload(q, p)
    one.advance(2)
    one.sync()
    wq, wp = one.download()
    if backend == EXACT:
        gs.set_exact_pairs(-1)
        assert gs.exact_pairs_plan(n, F32) > 0
        sym = gs.flow(cfg, n)
        sym.upload(q, p)
        sym.advance(2)
        sym.sync()
        sq, sp = sym.download()
        assert rel_l2(sq, wq) < 1e-6 and rel_l2(sp, wp) < 1e-5
        gs.set_exact_pairs(1)

    a, b = gs.flow(cfg, n), gs.flow(cfg, n)
    for f in (a, b):
        f.upload(q, p)
    h = n // 2
    a.set_shard(0, h)
    b.set_shard(h, n - h)
    ra, rb = records_view(a), records_view(b)
    per = ra.numel() // n
    for _ in range(2):
        for s in range(4):
            a.stage(s)
            b.stage(s)
            torch.cuda.synchronize()
            ra[h * per:] = rb[h * per:]
            rb[:h * per] = ra[:h * per]
            torch.cuda.synchronize()
    for f in (a, b):
        f.sync()
    for f in (a, b):
        gq, gp = f.download()
        if backend == EXACT:  # shards run the full problem's launch plan: bit-identical
            assert np.array_equal(gq, wq) and np.array_equal(gp, wp)
        else:  # same interaction sets; the group walk's summation order depends on the warp
            assert rel_l2(gq, wq) < 1e-6 and rel_l2(gp, wp) < 1e-5
