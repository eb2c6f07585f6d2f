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
from paper_1907_04834_b200.shard import _CudaBuf, records_view
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


def _pair_shards(gs, q, p, cfg, world, steps):
    """Symmetric multi-GPU stages emulated with `world` flows on one GPU: each
    evaluates its rows of the tile-pair grid, the per-target partials are
    exchanged as the all-to-all of shard.ShardedFlow would (rank r receives
    every rank's slice of its shard, in rank order), each shard's epilogue
    folds them, and the updated records are exchanged."""
    n = len(q)
    flows = [gs.flow(cfg, n) for _ in range(world)]
    cnt = n // world
    for r, f in enumerate(flows):
        f.upload(q, p)
        f.set_shard(r * cnt, cnt)
        assert f.set_pair_rows(r, world)
    recs = [records_view(f) for f in flows]
    per = recs[0].numel() // n
    outs = [torch.empty(world * cnt * 8, dtype=torch.float32, device="cuda") for _ in range(world)]
    stages = 4 if cfg.integrator == RK4 else 1
    for _ in range(steps):
        for s in range(stages):
            parts = []
            for f in flows:
                ptr = f.stage_pairs(s)
                torch.cuda.synchronize()
                parts.append(torch.as_tensor(_CudaBuf(ptr, n * 32), device="cuda").clone())
            for r, f in enumerate(flows):
                for w in range(world):
                    outs[r][w * cnt * 8:(w + 1) * cnt * 8] = parts[w][r * cnt * 8:(r + 1) * cnt * 8]
                torch.cuda.synchronize()
                f.stage_apply(s, outs[r].data_ptr(), world)
            torch.cuda.synchronize()
            for r in range(world):
                for w in range(world):
                    if w != r:
                        recs[w][r * cnt * per:(r + 1) * cnt * per] = recs[r][r * cnt * per:(r + 1) * cnt * per]
            torch.cuda.synchronize()
    for f in flows:
        f.sync()
    return [f.download() for f in flows]


def test_pair_rows_shards_match_one_flow(gs):
    """Symmetric multi-GPU stages (gs_flow_set_pair_rows): 1 rank is bitwise
    the one-GPU symmetric flow (its fold takes every slot in slot order); 2 and
    3 ranks (3: unequal row counts) equal it to FP32 rounding and are bitwise
    repeatable."""
    n = 60_000
    rng = np.random.default_rng(78)
    q, p = rng.uniform(0, 1, (n, 3)), rng.normal(0, 1e-2, (n, 3))
    cfg = ShootingConfig(sigma=0.03, timesteps=10, backend=EXACT, integrator=RK4, precision=F32)
    assert gs.exact_pairs_plan(n, F32) > 0
    one = gs.flow(cfg, n)
    one.upload(q, p)
    one.advance(2)
    one.sync()
    wq, wp = one.download()
    (aq, ap), = _pair_shards(gs, q, p, cfg, 1, 2)
    assert np.array_equal(aq, wq) and np.array_equal(ap, wp)
    for world in (2, 3):
        got = _pair_shards(gs, q, p, cfg, world, 2)
        again = _pair_shards(gs, q, p, cfg, world, 2)
        for (gq, gp), (hq, hp) in zip(got, again):
            assert np.array_equal(gq, hq) and np.array_equal(gp, hp)
            assert rel_l2(gq, wq) < 1e-6 and rel_l2(gp, wp) < 1e-5


def test_pair_rows_not_for_gather_problems(gs):
    cfg = ShootingConfig(sigma=0.03, timesteps=10, backend=EXACT, integrator=RK4, precision=F32)
    f = gs.flow(cfg, 5_000)  # below 8k points: the gather kernel
    assert not f.set_pair_rows(0, 2)
    fb = gs.flow(ShootingConfig(sigma=0.03, timesteps=10, backend=BARNES_HUT, precision=F32), 60_000)
    assert not fb.set_pair_rows(0, 2)


def _nccl_single_rank(out):
    import os
    import torch.distributed as dist
    from paper_1907_04834_b200 import Geoshoot
    from paper_1907_04834_b200.shard import ShardedFlow
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(29900 + os.getpid() % 90)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    gs = Geoshoot(0)
    n = 40_000
    rng = np.random.default_rng(79)
    q, p = rng.uniform(0, 1, (n, 3)), rng.normal(0, 1e-4, (n, 3))
    cfg = ShootingConfig(sigma=0.03, timesteps=10, backend=EXACT, integrator=RK4, precision=F32)
    f = gs.flow(cfg, n)
    drv = ShardedFlow(f, 4, pairs=True)
    assert drv.pairs
    f.upload(q, p)
    drv.step(2)
    f.sync()
    gq, gp = f.download()
    one = gs.flow(cfg, n)
    one.upload(q, p)
    one.advance(2)
    one.sync()
    wq, wp = one.download()
    np.savez(out, gq=gq, gp=gp, wq=wq, wp=wp, coll=drv.collectives)
    dist.destroy_process_group()


def test_pair_rows_through_nccl_single_rank(tmp_path):
    """The torchrun path's pair-row stages through a real NCCL process group
    (one rank on one GPU: the all-to-all is a copy): the ShardedFlow stage
    sequence -- gs_flow_stage_pairs on the flow's stream, all_to_all_single on
    that stream, gs_flow_stage_apply, the record all-gather -- bitwise equal to
    the one-GPU symmetric flow (a one-rank fold takes every slot in order)."""
    import torch.multiprocessing as mp
    out = str(tmp_path / "nccl1.npz")
    ctx = mp.get_context("spawn")
    proc = ctx.Process(target=_nccl_single_rank, args=(out,))
    proc.start()
    proc.join(600)
    assert proc.exitcode == 0
    d = np.load(out)
    assert int(d["coll"]) == 8  # 2 steps x 4 stages x all-to-all (no all-gather with one rank)
    assert np.array_equal(d["gq"], d["wq"]) and np.array_equal(d["gp"], d["wp"])
