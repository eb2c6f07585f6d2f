#!/usr/bin/env python
"""Benchmark of the B200 geodesic-shooting hot path (BASELINE.json metric:
"flow steps/s & G pair-interactions/s at N=100k-1M; % of FP32/SFU roofline").

Workload (BASELINE config 4, the configuration the metric is quoted on, the
largest that fits one GPU): N = 1,000,000 points uniform i.i.d. in the unit
cube, momenta i.i.d. N(0, 1e-4) per component (variance 1e-4), sigma = 0.0131,
FP32, RK4 with 10 steps over [0, 1] (dt = 0.1), exact all-pairs kernel. One
bench "step" = one RK4 flow step = 4 exact right-hand sides = 4 N^2 ordered
pair interactions. The same flow through the Barnes-Hut back end (3 sigma
gate, tree rebuilt at every stage) is reported under "bh".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--n N]

Multi-GPU (torchrun, one rank per GPU): targets are sharded across ranks and
the updated (q, p) records are all-gathered over NCCL after every stage
(paper_1907_04834_b200/shard.py); time = max over ranks of the device time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SIGMA = 0.0131
T_STEPS = 10
METRIC = "flow steps/s (RK4, 4 RHS/step) & G pair-interactions/s, config 4"
# Algorithmic DRAM bytes per point of one FP32 tree build (DESIGN.md §4 table)
BUILD_BYTES_PER_POINT = 1080


def workload(n: int, seed: int = 2024):
    rng = np.random.default_rng(seed)
    q = rng.uniform(0.0, 1.0, (n, 3))
    p = rng.normal(0.0, 1e-2, (n, 3))  # N(0, 1e-4): variance 1e-4
    return q, p


def peaks_json():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) > 2 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 2 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows if len(r) >= 9 for k in range(4)
                          if r[5 + k].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------
def cpu_reference(n_sample: int, threads: int, reps: int = 1):
    """The reference's own exact RHS (kernel_exact.cpp:29-61, compiled by path
    into oracle/_ref) on `threads` host threads concurrently, each on the same
    n_sample-point input. Returns ordered pair interactions per second."""
    import oracle
    R = oracle.ref() if oracle.have_ref() else None
    q, p = workload(n_sample, seed=7)
    t0 = time.perf_counter()
    if R is not None:
        R.exact_rhs_concurrent(q, p, SIGMA, threads, reps)
        kind = "reference"
    else:  # the C restatement (oracle/port.c), serial
        for _ in range(reps):
            oracle.port().exact_rhs(q, p, SIGMA)
        threads, kind = 1, "port"
    dt = time.perf_counter() - t0
    return threads * reps * float(n_sample) ** 2 / dt, threads, kind


def run_reference(args):
    """--impl reference: the reference CPU implementation of the path, all host threads."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n_s = args.cpu_sample
    rates = []
    for k in range(args.warmup + args.steps):
        r, used, kind = cpu_reference(n_s, threads)
        if k >= args.warmup:
            rates.append(r)
    rate = float(np.mean(rates))
    value = rate / (4.0 * float(args.n) ** 2)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "flow steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 / value, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config4 exact RK4 N={args.n} (extrapolated by N^2 from a sample)",
                   "n": args.n, "sigma": SIGMA, "integrator": "rk4", "timesteps": T_STEPS},
        "pair_interactions_per_s": rate,
        "cpu_baseline": {"value": value, "unit": "flow steps/s", "cores": used, "kind": kind,
                         "sample": f"{used} concurrent reference hamiltonian_gradients calls at "
                                   f"N={n_s} per step ({n_s}^2 ordered pairs each), extrapolated "
                                   f"to N={args.n} by N^2 x 4 RHS/step"},
        "e2e": {"value": value, "unit": "flow steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1907_04834_b200 import BARNES_HUT, EXACT, F32, RK4, Geoshoot, ShootingConfig
    from paper_1907_04834_b200 import _lib
    from paper_1907_04834_b200.shard import ShardedFlow

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")
    N = args.n
    q0, p0 = workload(N)

    gs = Geoshoot(local)
    cfg = ShootingConfig(sigma=SIGMA, timesteps=T_STEPS, backend=EXACT, integrator=RK4,
                         precision=F32)
    flow = gs.flow(cfg, N)
    flow.upload(q0, p0)
    stream = torch.cuda.ExternalStream(flow.stream())
    drv = ShardedFlow(flow, 4, stream=stream) if world > 1 else None
    shard = N // world

    def step():
        if drv is None:
            flow.advance(1)
        else:
            drv.step(1)

    # L2 is 126 MB and the records are 32 MB: flush it before every timed step
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    flow.sync()
    barrier()
    flow.profile(True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks = Clocks(local)
    launches = 0
    barrier()
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
        launches += flow.last_launches() if drv is None else 8
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    flow.sync()  # raises NonFiniteState if the flow blew up
    ms = sum(a.elapsed_time(b) for a, b in ev)
    prof = flow.profile_read()
    flow.profile(False)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = args.steps / (ms / 1e3)
    pairs_per_s = 4.0 * N * float(N) * args.steps / (ms / 1e3)

    # roofline of the dominant kernel (all-pairs RHS): issue-bound at 16 FP32
    # instructions per pair; peak from a live FFMA microbenchmark
    lib = _lib.load()
    import ctypes as C
    ffma = C.c_double()
    lib.gs_microbench(local, 0, C.byref(ffma))
    ex2 = C.c_double()
    lib.gs_microbench(local, 1, C.byref(ex2))
    ffma_reg = C.c_double()
    lib.gs_microbench(local, 3, C.byref(ffma_reg))
    ffma2 = C.c_double()
    lib.gs_microbench(local, 4, C.byref(ffma2))
    k_ms = prof["kernel_ms"] / max(1, prof["kernel_launches"])
    pairs_per_launch = float(N) * shard
    achieved = pairs_per_launch / (k_ms * 1e-3) / 1e9  # Gpair/s
    peak = ffma.value / 16.0 / 1e9
    mp = peaks_json()
    nominal = 148 * 128 * float(mp.get("sm_max_mhz", 1965.0)) * 1e6 / 16.0 / 1e9
    traffic = None
    try:  # dram bytes per launch of the same kernel from the committed ncu capture
        tj = json.load(open(os.path.join(ROOT, "profiles", "r01_rhs_traffic.json")))
        if tj.get("n") == N and world == 1:
            traffic = tj["dram_bytes_per_launch"]
    except Exception:
        pass
    roofline = {
        "bound": "fp32-issue", "achieved": achieved, "peak": peak, "unit": "Gpair/s",
        "frac": achieved / peak, "traffic": traffic,
        "traffic_unit": "DRAM bytes per launch (ncu, profiles/r01_rhs_traffic.json)",
        "peak_source": "live FFMA microbenchmark (gs_microbench kind 0): "
                       f"{ffma.value / 1e12:.2f} T lane-FFMA/s / 16 FP32 instructions per pair; "
                       "MEASURED_PEAKS.json has no FP32 figure",
        "nominal_peak": nominal, "frac_of_nominal": achieved / nominal,
        "peak_register_operand_ffma": ffma_reg.value / 16.0 / 1e9,
        "peak_packed_ffma2": ffma2.value / 16.0 / 1e9,
        "sfu_frac": achieved * 1e9 / ex2.value if ex2.value else None,
        "kernel": "k_rhs_f32x2<12,128,2,8> (packed FFMA2, source loop unrolled 8)", "kernel_ms_avg": k_ms,
        "kernel_share_of_step": prof["kernel_ms"] / ms if ms else None,
        "algorithmic_per_launch": f"{pairs_per_launch:.3e} ordered pairs x 16 FP32 + 1 MUFU",
    }

    line = {
        "metric": METRIC, "value": value, "unit": "flow steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded uniform cube, BASELINE config 4)",
        "config": {"workload": f"config4: exact all-pairs RHS, RK4 x {T_STEPS} steps, N={N}, "
                               f"sigma={SIGMA}, unit cube, fp32; 1 step = 4 RHS",
                   "n": N, "sigma": SIGMA, "integrator": "rk4", "timesteps": T_STEPS,
                   "backend": "exact", "parallelism": f"target-shard x{world}",
                   "l2": "flushed (256 MB write) before every timed step"},
        "pair_interactions_per_s": pairs_per_s,
        "gpu_launches": launches,
        "clocks": clk,
        "roofline": roofline,
    }

    # ---- Barnes-Hut back end on the same workload (rank 0 reporting) -----------
    if not args.no_bh and world == 1:
        cfg_bh = ShootingConfig(sigma=SIGMA, timesteps=T_STEPS, backend=BARNES_HUT,
                                integrator=RK4, precision=F32)
        fb = gs.flow(cfg_bh, N)
        fb.upload(q0, p0)
        sb = torch.cuda.ExternalStream(fb.stream())
        fb.advance(max(1, args.warmup))
        fb.sync()
        # time the first kb steps of the config-4 flow itself (the point
        # distribution, hence the traversal work, evolves along the flow)
        fb.upload(q0, p0)
        fb.sync()
        st0 = fb.stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kb = max(1, args.steps)
        with torch.cuda.stream(sb):
            flush.zero_()
        e0.record(sb)
        fb.advance(kb)  # production path: steps after the first replay a CUDA graph
        e1.record(sb)
        torch.cuda.synchronize()
        fb.sync()
        bms = e0.elapsed_time(e1)
        st1 = fb.stats()
        # per-phase kernel times: the same steps again, profiled (eager launches)
        fb.upload(q0, p0)
        fb.sync()
        fb.profile(True)
        fb.advance(kb)
        fb.sync()
        ph = fb.profile_phases(6)
        fb.profile(False)
        rhs = 4 * kb
        d = st1["direct_interactions"] - st0["direct_interactions"]
        a_ = st1["approximated_interactions"] - st0["approximated_interactions"]
        v = st1["nodes_visited"] - st0["nodes_visited"]
        trav_s = ph["kernel"]["ms"] / 1e3
        build_ms = ph["build"]["ms"] / max(1, ph["build"]["count"])
        lane_peak = ffma.value  # lane FFMA/s (live microbenchmark)
        line["bh"] = {
            "value": kb / (bms / 1e3), "unit": "flow steps/s", "ms_per_step": bms / kb,
            "n2_equivalent_pairs_per_s": 4.0 * N * float(N) * kb / (bms / 1e3),
            "interactions_per_s": (d + a_) / (bms / 1e3),
            "per_query_per_rhs": {"direct": d / (rhs * N), "approximated": a_ / (rhs * N),
                                  "visited": v / (rhs * N)},
            "traversal_ms_per_rhs": ph["kernel"]["ms"] / max(1, ph["kernel"]["count"]),
            "tree_build_ms_per_rhs": build_ms,
            "build_phases_ms_per_rhs": {k: ph[k]["ms"] / max(1, ph[k]["count"])
                                        for k in ("bbox_keys", "sort", "topology", "aggregate")},
            # 16 FP32 per interaction + 12 per visited node
            "traversal_fp32_issue_frac": ((16.0 * (d + a_) + 12.0 * v) / trav_s) / lane_peak
            if trav_s > 0 else None,
            # algorithmic bytes of the build kernels, FP32 (per point)
            "build_gbs_algorithmic": BUILD_BYTES_PER_POINT * N / (build_ms * 1e-3) / 1e9,
            "build_hbm_frac": BUILD_BYTES_PER_POINT * N / (build_ms * 1e-3) / 1e9
            / float(mp.get("hbm_gbs", 6550.0)),
            "kernel": "k_bh_ws<float> (independent walks); tree: radix sort + LCP topology",
        }
        del fb

    # ---- Barnes-Hut across ranks: target shards (Morton-ordered at set_shard),
    # one in-place all-gather per stage; device time = max over ranks ----------
    def bh_sharded():
        cfg_bh = ShootingConfig(sigma=SIGMA, timesteps=T_STEPS, backend=BARNES_HUT,
                                integrator=RK4, precision=F32)
        fb = gs.flow(cfg_bh, N)
        fb.upload(q0, p0)
        sb = torch.cuda.ExternalStream(fb.stream())
        drb = ShardedFlow(fb, 4, stream=sb)
        drb.step(max(1, args.warmup))
        fb.sync()
        # time the first kb steps of the config-4 flow (as on one GPU): re-upload,
        # re-shard (Morton order again, fresh record view)
        fb.upload(q0, p0)
        drb = ShardedFlow(fb, 4, stream=sb)
        barrier()
        kb = max(1, args.steps)
        with torch.cuda.stream(sb):
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sb)
        drb.step(kb)
        e1.record(sb)
        torch.cuda.synchronize()
        barrier()
        fb.sync()
        t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        bms = float(t.item())
        line["bh"] = {"value": kb / (bms / 1e3), "unit": "flow steps/s", "ms_per_step": bms / kb,
                      "n2_equivalent_pairs_per_s": 4.0 * N * float(N) * kb / (bms / 1e3),
                      "parallelism": f"target-shard x{world} (each rank rebuilds the tree)"}
        del drb, fb

    if not args.no_bh and world > 1:
        try:  # an auxiliary line: never let it take the headline down
            bh_sharded()
        except Exception as exc:  # noqa: BLE001
            line["bh"] = {"error": f"{type(exc).__name__}: {exc}"}

    # ---- exact with the FP32 underflow cutoff (GS_FLAG_EXACT_CUTOFF, opt-in) ------
    # The same exact sum over Morton-ordered points, skipping tile pairs whose
    # Gaussian weights are all exactly 0 in FP32 (bit-identical to evaluating
    # them in that order; tests/test_gpu_exact.py). Not the headline: the
    # headline `value` evaluates all N^2 pairs.
    if not args.no_extra and world == 1:
        cfg_c = ShootingConfig(sigma=SIGMA, timesteps=T_STEPS, backend=EXACT, integrator=RK4,
                               precision=F32, exact_cutoff=True)
        fc = gs.flow(cfg_c, N)
        sc = torch.cuda.ExternalStream(fc.stream())
        fc.upload(q0, p0)
        fc.advance(max(1, args.warmup))
        fc.sync()
        fc.upload(q0, p0)  # time the first steps of the config-4 flow
        fc.sync()
        kc_ = max(1, args.steps)
        with torch.cuda.stream(sc):
            flush.zero_()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(sc)
        fc.advance(kc_)
        c1.record(sc)
        torch.cuda.synchronize()
        fc.sync()
        cms = c0.elapsed_time(c1)
        line["exact_cutoff"] = {
            "value": kc_ / (cms / 1e3), "unit": "flow steps/s", "ms_per_step": cms / kc_,
            "speedup_vs_all_pairs": (kc_ / (cms / 1e3)) / value,
            "note": "exact FP32 sum in Morton order; (target group, source tile) pairs beyond "
                    "the FP32 underflow radius of 2^-r'^2 skipped (their terms are exactly 0)",
        }
        del fc

    # ---- exact FP64 and N = 100k FP32 lines (same workload family) -------------
    if not args.no_extra and world == 1:
        def timed_flow(n, prec, integ, steps):
            qq, pp = workload(n)
            c = ShootingConfig(sigma=SIGMA, timesteps=T_STEPS, backend=EXACT, integrator=integ,
                               precision=prec)
            fl = gs.flow(c, n)
            fl.upload(qq, pp)
            s_ = torch.cuda.ExternalStream(fl.stream())
            fl.advance(1)
            fl.sync()
            fl.profile(True)
            t0_, t1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0_.record(s_)
            fl.advance(steps)
            t1_.record(s_)
            torch.cuda.synchronize()
            fl.sync()
            pr = fl.profile_read()
            return t0_.elapsed_time(t1_), pr
        from paper_1907_04834_b200 import EULER, F64
        n64 = 200_000
        ms64, pr64 = timed_flow(n64, F64, EULER, 2)
        dfma = C.c_double()
        lib.gs_microbench(local, 2, C.byref(dfma))
        k64 = pr64["kernel_ms"] / max(1, pr64["kernel_launches"])
        pps64 = float(n64) * n64 / (k64 * 1e-3)
        line["fp64"] = {
            "workload": f"exact FP64 RHS, N={n64}, Euler (config-4 distribution)",
            "pair_interactions_per_s": pps64, "kernel_ms": k64,
            "steps_per_s": 2 / (ms64 / 1e3),
            "peak_dfma_lane_per_s": dfma.value,
            "frac_16dp_basis": pps64 * 16.0 / dfma.value if dfma.value else None,
            # + the 10-DP table-driven exp of the FP64 kernels (csrc/gs_exp.cuh)
            "frac_26dp_basis_incl_exp": pps64 * 26.0 / dfma.value if dfma.value else None,
        }
        ms1, pr1 = timed_flow(100_000, F32, RK4, 3)
        line["n100k"] = {
            "value": 3 / (ms1 / 1e3), "unit": "flow steps/s (RK4)",
            "pair_interactions_per_s": 4.0 * 1e10 * 3 / (ms1 / 1e3),
            "frac_of_ffma_peak": (4.0 * 1e10 * 3 / (ms1 / 1e3)) / peak / 1e9,
        }

    # ---- end to end through the public C-ABI call, host buffers ----------------
    if world == 1:
        pin_q = torch.empty((N, 3), dtype=torch.float64, pin_memory=True).numpy()
        pin_p = torch.empty((N, 3), dtype=torch.float64, pin_memory=True).numpy()
        pin_q[:] = q0
        pin_p[:] = p0
        t0 = time.perf_counter()
        fq, fp, energy, _ = gs.shoot_forward(pin_q, pin_p, cfg, keep_trajectory=False)
        dt = time.perf_counter() - t0
        line["e2e"] = {"value": T_STEPS / dt, "unit": "flow steps/s",
                       "h2d_bytes_per_step": 2 * N * 24 // T_STEPS,
                       "d2h_bytes_per_step": 2 * N * 24 // T_STEPS,
                       "call": f"gs_shoot_forward (10 RK4 steps, final state only) x1, {dt:.2f} s"}

    # ---- CPU baseline: the reference's own exact RHS on the host cores ---------
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        rate, used, kind = cpu_reference(args.cpu_sample, threads)
        line["cpu_baseline"] = {
            "value": rate / (4.0 * float(N) ** 2), "unit": "flow steps/s", "cores": used,
            "kind": kind, "pair_interactions_per_s": rate,
            "sample": f"{used} concurrent reference hamiltonian_gradients calls at N={args.cpu_sample} "
                      f"(FP64, serial by construction per call), extrapolated to N={N} by N^2 x 4 RHS/step"}
        if "bh" in line and kind == "reference":
            # the reference's Barnes-Hut path on the same flow: one Euler step of
            # shoot_forward (serial octree build + one parallel_for RHS,
            # bh_kernel.cpp:193-210) at the full N; an RK4 step is 4 of them
            import oracle
            t0 = time.perf_counter()
            oracle.ref().shoot_forward(q0, p0, SIGMA, 1, backend=1)
            t_rhs = time.perf_counter() - t0
            line["bh"]["cpu_baseline"] = {
                "value": 1.0 / (4.0 * t_rhs), "unit": "flow steps/s", "cores": threads,
                "kind": "reference", "seconds_per_rhs": t_rhs,
                "sample": f"reference shoot_forward, Barnes-Hut, T=1 (one tree build + one RHS) at "
                          f"N={N}, FP64, GEOSHOOT_THREADS default ({threads} host threads); x4 RHS per RK4 step"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--cpu-sample", type=int, default=8192)
    ap.add_argument("--no-extra", action="store_true", help="skip the FP64 / N=100k lines")
    ap.add_argument("--no-bh", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
