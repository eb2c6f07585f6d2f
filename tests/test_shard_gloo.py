"""World-size-2 CPU test (gloo) of the multi-GPU driver (paper_1907_04834_b200/shard.py).

The device flow is replaced by a CPU stand-in with the same stage/shard/record
interface whose RHS is the CPU oracle (test infrastructure only); the driver
code under test -- shard ranges, in-place all-gather of the updated records
after every stage -- is the one bench.py runs over NCCL on B200s. Sharded
results must be bitwise identical to the unsharded run.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1907_04834_b200.shard import ShardedFlow, register_subjects, shard_range, subject_range


class CpuFlow:
    """Stand-in flow: FP64 records [n][2][4] (q, 0, p, 0), Euler stages."""

    def __init__(self, q, p, sigma, dt):
        import oracle
        self.port = oracle.port()
        self.n = len(q)
        rec = np.zeros((self.n, 2, 4))
        rec[:, 0, :3], rec[:, 1, :3] = q, p
        self.rec = torch.from_numpy(rec.reshape(-1).copy())
        self.sigma, self.dt = sigma, dt
        self.begin, self.count = 0, self.n

    def records(self):
        return self.rec

    def set_shard(self, begin, count):
        self.begin, self.count = begin, count

    def stage(self, s):
        r = self.rec.numpy().reshape(self.n, 2, 4)
        dp, dq, _ = self.port.exact_rhs(r[:, 0, :3], r[:, 1, :3], self.sigma)
        sl = slice(self.begin, self.begin + self.count)
        r[sl, 0, :3] += self.dt * dp[sl]
        r[sl, 1, :3] -= self.dt * dq[sl]

    def state(self):
        r = self.rec.numpy().reshape(self.n, 2, 4)
        return r[:, 0, :3].copy(), r[:, 1, :3].copy()


class PairCpuFlow(CpuFlow):
    """Stand-in for the symmetric multi-GPU stages (gs_flow_set_pair_rows):
    tiles of 8 points, rank r evaluates the unordered tile pairs of its rows
    (CTA (I, k), J = (I + k) mod T, k = 0..T/2, the even-T k = T/2 pairs by
    I < T/2 only -- allpairs.cu k_rhs_sym_f32x2) for BOTH ends, folds them per
    target, and the shard's epilogue folds the world partials it receives."""
    TILE = 8

    def set_pair_rows(self, rank, world):
        self.rank, self.world = rank, world
        return True

    def stage_pairs_tensor(self, s):
        r = self.rec.numpy().reshape(self.n, 2, 4)
        q, p = r[:, 0, :3], r[:, 1, :3]
        T = (self.n + self.TILE - 1) // self.TILE
        ra, rb = T * self.rank // self.world, T * (self.rank + 1) // self.world
        A, B = np.zeros((self.n, 3)), np.zeros((self.n, 3))
        inv = 1.0 / (2 * self.sigma ** 2)

        def add(ti, tj):  # targets of tile ti from sources of tile tj
            a, b = slice(ti * self.TILE, (ti + 1) * self.TILE), slice(tj * self.TILE, (tj + 1) * self.TILE)
            d = q[a][:, None, :] - q[b][None, :, :]
            g = np.exp(-(d * d).sum(2) * inv)
            A[a] += g @ p[b]
            B[a] += ((p[a] @ p[b].T) * g)[:, :, None].__mul__(d).sum(1)

        for I in range(ra, rb):
            for k in range(T // 2 + 1):
                if 2 * k == T and I >= k:
                    continue
                J = (I + k) % T
                add(I, J)
                if k:
                    add(J, I)
        out = np.zeros((self.n, 8))
        out[:, :3], out[:, 4:7] = A, B
        return torch.from_numpy(out.reshape(-1).copy())

    def stage_apply_tensor(self, s, parts, world):
        x = parts.numpy().reshape(world, self.count, 8)
        A, B = x[0, :, :3].copy(), x[0, :, 4:7].copy()
        for w in range(1, world):
            A += x[w, :, :3]
            B += x[w, :, 4:7]
        r = self.rec.numpy().reshape(self.n, 2, 4)
        sl = slice(self.begin, self.begin + self.count)
        r[sl, 0, :3] += self.dt * 2.0 * A            # dH/dp = 2 sum g p
        r[sl, 1, :3] -= self.dt * (-2.0 / self.sigma ** 2) * B  # dH/dq = -(2/s) sum c d


def inputs():
    rng = np.random.default_rng(5)
    return rng.uniform(0, 2, (64, 3)), rng.uniform(-0.3, 0.3, (64, 3))


def worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q, p = inputs()
    f = CpuFlow(q, p, 0.7, 0.1)
    drv = ShardedFlow(f, stages=1)
    assert (drv.begin, drv.count) == shard_range(64, rank, world)
    drv.step(5)
    fq, fp = f.state()
    np.save(os.path.join(out, f"q{rank}.npy"), fq)
    np.save(os.path.join(out, f"p{rank}.npy"), fp)
    assert drv.collectives == 5
    dist.destroy_process_group()


def test_shard_ranges():
    assert shard_range(1_000_000, 3, 8) == (375_000, 125_000)
    with pytest.raises(ValueError):
        shard_range(10, 0, 3)


def test_two_rank_gloo_matches_single_rank(tmp_path):
    port = 29500 + os.getpid() % 1000
    mp.spawn(worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    q, p = inputs()
    f = CpuFlow(q, p, 0.7, 0.1)
    for _ in range(5):
        f.stage(0)
    wq, wp = f.state()
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"q{r}.npy"), wq)
        assert np.array_equal(np.load(tmp_path / f"p{r}.npy"), wp)


def fake_batch(templates, targets, cfg, **opt):
    """CPU stand-in for Geoshoot.optimize_batch: a deterministic per-subject result."""
    return {"p0": [0.5 * (t - q) for q, t in zip(templates, targets)],
            "reasons": [1] * len(templates), "iterations": [len(q) for q in templates],
            "evaluations": [len(q) + 1 for q in templates],
            "final_total": np.array([float(np.abs(t - q).sum()) for q, t in zip(templates, targets)])}


def subjects():
    rng = np.random.default_rng(11)
    qs = [rng.uniform(0, 1, (5 + k, 3)) for k in range(7)]
    ts = [q + 0.1 * (k + 1) for k, q in enumerate(qs)]
    return qs, ts


def subject_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    qs, ts = subjects()
    seen = []

    def runner(a, b, cfg, **opt):
        seen.append(len(a))
        return fake_batch(a, b, cfg, **opt)

    res = register_subjects(None, qs, ts, cfg=None, runner=runner, max_iterations=3)
    assert seen == [subject_range(7, rank, world)[1]]
    np.save(os.path.join(out, f"s{rank}.npy"),
            np.concatenate([np.concatenate([[r["subject"], r["iterations"], r["final_total"]],
                                            r["p0"].ravel()]) for r in res]))
    dist.destroy_process_group()


def test_subject_ranges_cover_all():
    for count in (0, 1, 7, 64):
        for world in (1, 2, 3, 8):
            spans = [subject_range(count, r, world) for r in range(world)]
            assert sum(c for _, c in spans) == count
            assert all(spans[r][0] + spans[r][1] == spans[r + 1][0] for r in range(world - 1))


def test_two_rank_subjects_match_single_rank(tmp_path):
    port = 29600 + os.getpid() % 1000
    mp.spawn(subject_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    qs, ts = subjects()
    want = register_subjects(None, qs, ts, cfg=None, runner=fake_batch)
    flat = np.concatenate([np.concatenate([[r["subject"], r["iterations"], r["final_total"]],
                                           r["p0"].ravel()]) for r in want])
    assert [r["subject"] for r in want] == list(range(7))
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"s{r}.npy"), flat)


def pair_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q, p = inputs()
    f = PairCpuFlow(q, p, 0.7, 0.1)
    drv = ShardedFlow(f, stages=1)
    assert drv.pairs
    drv.step(5)
    assert drv.collectives == 10  # all-to-all of the partials + all-gather of the records
    fq, fp = f.state()
    np.save(os.path.join(out, f"q{rank}.npy"), fq)
    np.save(os.path.join(out, f"p{rank}.npy"), fp)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_pair_rows_gloo_match_single_rank(tmp_path, world):
    """The symmetric multi-GPU stage logic (rows of the tile-pair grid, the
    all-to-all of per-target partials, the shard epilogue) over gloo against
    the unsharded reference-RHS flow: every unordered pair exactly once
    (T = 8 tiles: even T, so the k = T/2 rule matters)."""
    port = 29700 + world * 10 + os.getpid() % 500
    mp.spawn(pair_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    q, p = inputs()
    f = CpuFlow(q, p, 0.7, 0.1)
    for _ in range(5):
        f.stage(0)
    wq, wp = f.state()
    for r in range(world):
        assert np.allclose(np.load(tmp_path / f"q{r}.npy"), wq, rtol=0, atol=1e-12)
        assert np.allclose(np.load(tmp_path / f"p{r}.npy"), wp, rtol=0, atol=1e-12)
