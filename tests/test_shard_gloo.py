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

from paper_1907_04834_b200.shard import ShardedFlow, shard_range


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
