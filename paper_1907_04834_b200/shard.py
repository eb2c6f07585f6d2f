"""Multi-GPU driver: target sharding with one all-gather per integrator stage.

SURVEY.md §8e: within a stage every target's RHS is independent, so rank r
owns targets [r*N/G, (r+1)*N/G), computes their RHS against all N sources and
updates its own records in the fused stage epilogue; then the ranks all-gather
the updated shards (torch.distributed, NCCL over NVLink/NVSwitch on B200s,
gloo in the CPU tests). The all-gather is in place: every rank's record buffer
is the gather output and its own shard is the input slice. An exact shard
launches under the full problem's plan (gs_flow_set_shard), so its per-target
sums -- and the flow -- are bit-identical to one GPU's gather-kernel run
(below 8k points the one-GPU default; above it one GPU takes the symmetric
kernel, equal to FP32 rounding -- DESIGN.md §2, §7); Barnes-Hut shards have
the reference's interaction sets, equal to summation-order rounding.

(Inside ONE process, gs_create_multi / Geoshoot(devices=[...]) shards across
devices without torch.distributed: the exchange is fused into the stage
epilogues as P2P stores.)
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def subject_range(count: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of independent subjects for a rank (any count: the
    first count % world ranks take one extra)."""
    base, extra = divmod(count, world)
    begin = rank * base + min(rank, extra)
    return begin, base + (1 if rank < extra else 0)


def register_subjects(gs, templates, targets, cfg, group=None, runner=None, **opt):
    """Config 5 across GPUs (SURVEY.md §8e "batched subjects"): independent
    registrations, no data-path collective. Rank r optimises its contiguous
    block of subjects concurrently on its own GPU (``Geoshoot.optimize_batch``:
    one stream + host thread per subject) and the per-subject results are
    gathered to every rank once at the end (``all_gather_object``: O(subjects)
    small host objects plus the p0 arrays). Results are bitwise the ones a
    single GPU computes for the same subjects.

    ``runner(templates, targets, cfg, **opt)`` defaults to ``gs.optimize_batch``
    (tests substitute a CPU stand-in). Returns the list of per-subject dicts
    {"subject", "p0", "reason", "iterations", "evaluations", "final_total"} in
    subject order.
    """
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    b, c = subject_range(len(templates), rank, world)
    run = runner if runner is not None else gs.optimize_batch
    mine = []
    if c:
        r = run(templates[b:b + c], targets[b:b + c], cfg, **opt)
        for k in range(c):
            mine.append({"subject": b + k, "p0": r["p0"][k], "reason": r["reasons"][k],
                         "iterations": r["iterations"][k], "evaluations": r["evaluations"][k],
                         "final_total": float(r["final_total"][k])})
    if world == 1:
        return mine
    parts = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    return [x for part in parts for x in part]


def evaluate_subjects(gs, templates, momenta, targets, cfg, group=None, runner=None):
    """Batched evaluations across ranks (SURVEY.md §8b ``gs_evaluate_batch``
    "distributed across ranks"): rank r evaluates its contiguous block of
    subjects concurrently on its GPU (``Geoshoot.evaluate_batch``) and the
    per-subject (report, gradient, stats) are gathered to every rank.
    Returns [{"subject", "report", "gradient", "stats"}] in subject order."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    b, c = subject_range(len(templates), rank, world)
    run = runner if runner is not None else gs.evaluate_batch
    mine = []
    if c:
        evs = run(templates[b:b + c], momenta[b:b + c], targets[b:b + c], cfg)
        mine = [{"subject": b + k, "report": e.report, "gradient": e.gradient, "stats": e.stats}
                for k, e in enumerate(evs)]
    if world == 1:
        return mine
    parts = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    return [x for part in parts for x in part]


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Equal contiguous shards (n must be divisible by world)."""
    if n % world:
        raise ValueError(f"point count {n} not divisible by world size {world}")
    s = n // world
    return rank * s, s


class _CudaBuf:
    """Exposes a raw device allocation to torch via __cuda_array_interface__."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {
            "shape": (nbytes // 4,), "typestr": "<f4", "data": (ptr, False), "version": 3,
            "strides": None}


def records_view(flow) -> torch.Tensor:
    """The flow's packed (q, p) records as a flat float32 CUDA tensor (no copy)."""
    nbytes = flow.n * flow.record_bytes()
    return torch.as_tensor(_CudaBuf(flow.source_buffer(), nbytes), device="cuda")


class ShardedFlow:
    """Drives a flow-like object over a torch.distributed process group.

    ``flow`` needs: n, stage(s), set_shard(begin, count), stages (int), and
    either a ``records()`` method returning its record tensor or the gs_flow
    accessors used by records_view(). ``stream`` (optional) is the CUDA stream
    the flow launches on; the all-gather is ordered after it.
    """

    def __init__(self, flow, stages: int, group=None, stream=None, pairs=None):
        self.flow = flow
        self.stages = stages
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.begin, self.count = shard_range(flow.n, self.rank, self.world)
        flow.set_shard(self.begin, self.count)
        if stream is None and hasattr(flow, "stream") and torch.cuda.is_available():
            # the flow launches on its own (non-blocking) stream: the gather must
            # be ordered after the stage epilogue and before the next stage
            stream = torch.cuda.ExternalStream(flow.stream())
        self.stream = stream
        self.launches = 0  # kernels of this rank's stages (gs_flow_last_launches)
        self._rec = flow.records() if hasattr(flow, "records") else records_view(flow)
        per = self._rec.numel() // flow.n
        self._mine = self._rec[self.begin * per:(self.begin + self.count) * per]
        self.collectives = 0
        # exact FP32 flows that take the symmetric kernel: each rank evaluates
        # its rows of the unordered tile-pair grid (both ends of every pair),
        # folds them per target, and the ranks exchange the shard slices of
        # those partials (all-to-all) before each shard's epilogue -- one
        # extra collective per stage, half the pair arithmetic of the gather
        # form
        # (pairs=True also takes the path with one rank: tests of the NCCL
        # exchange on a single GPU)
        want = (self.world > 1) if pairs is None else bool(pairs)
        self.pairs = (want and hasattr(flow, "set_pair_rows")
                      and flow.set_pair_rows(self.rank, self.world))
        if self.pairs:
            dev = self._rec.device
            self._pair_out = torch.empty(self.world * self.count * 8, dtype=self._rec.dtype, device=dev)

    def _pair_stage(self, s: int):
        """One symmetric stage: this rank's pair rows, the all-to-all of the
        per-target partials (rank r receives every rank's slice of its shard,
        in rank order) and the shard's epilogue over the world partials."""
        n = self.flow.n
        if hasattr(self.flow, "stage_pairs_tensor"):  # CPU stand-in (tests)
            inp = self.flow.stage_pairs_tensor(s)
        else:
            inp = torch.as_tensor(_CudaBuf(self.flow.stage_pairs(s), n * 32), device="cuda")
        if hasattr(self.flow, "last_launches"):
            self.launches += self.flow.last_launches()
        if self.stream is not None:
            with torch.cuda.stream(self.stream):
                dist.all_to_all_single(self._pair_out, inp, group=self.group)
        else:
            dist.all_to_all_single(self._pair_out, inp, group=self.group)
        self.collectives += 1
        if hasattr(self.flow, "stage_apply_tensor"):
            self.flow.stage_apply_tensor(s, self._pair_out, self.world)
        else:
            self.flow.stage_apply(s, self._pair_out.data_ptr(), self.world)
            if hasattr(self.flow, "last_launches"):
                self.launches += self.flow.last_launches()

    def _gather(self):
        if self.world == 1:
            return
        if self.stream is not None:
            with torch.cuda.stream(self.stream):
                dist.all_gather_into_tensor(self._rec, self._mine, group=self.group)
        else:
            dist.all_gather_into_tensor(self._rec, self._mine, group=self.group)
        self.collectives += 1

    def step(self, steps: int = 1):
        for _ in range(steps):
            for s in range(self.stages):
                if self.pairs:
                    self._pair_stage(s)
                else:
                    self.flow.stage(s)
                    if hasattr(self.flow, "last_launches"):
                        self.launches += self.flow.last_launches()
                self._gather()
