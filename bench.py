#!/usr/bin/env python
"""Benchmark of the B200 geodesic-shooting hot path (BASELINE.json metric:
"flow steps/s & G pair-interactions/s at N=100k-1M; % of FP32/SFU roofline").

Workload (BASELINE config 4, the configuration the metric is quoted on, the
largest that fits one GPU): N = 1,000,000 points uniform i.i.d. in the unit
cube, momenta i.i.d. N(0, 1e-4) per component (variance 1e-4), sigma = 0.0131,
FP32, RK4 with 10 steps over [0, 1] (dt = 0.1), exact all-pairs kernel. One
bench "step" = one RK4 flow step = 4 exact right-hand sides = 4 N^2 ordered
pair interactions (the exact kernel's cost does not depend on the positions).
Auxiliary lines on the same JSON line:

* ``bh``: the same flow through the Barnes-Hut back end (3 sigma gate, tree
  rebuilt at every stage), timed over exactly the config's 10 RK4 steps from
  q0 (a BH step's cost depends on the evolving positions);
* ``exact_cutoff``: the exact flow with the opt-in FP32 underflow cutoff, the
  same 10-step trajectory;
* ``adjoint``: config 3's unit of work -- one evaluate() (forward flow + kept
  trees + adjoint) at N = 50k, T = 20, FP32, exact and Barnes-Hut -- with the
  Hessian-product kernel's roofline;
* ``fp64``: one exact RK4 step at N = 1M in FP64 (the reference's precision:
  the like-for-like line against the FP64 reference CPU arm);
* ``n100k``; ``e2e`` (the public call with host buffers); ``cpu_baseline``.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--n N]

Multi-GPU (one process per GPU; ``--gpus N`` outside torchrun re-launches itself
under torch.distributed.run): targets are sharded across ranks and the updated
(q, p) records are all-gathered over NCCL after every stage
(paper_1907_04834_b200/shard.py); time = max over ranks of the device time.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import socket
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
# FP32 FMA-pipe operations per ordered pair
RHS_FP32_PER_PAIR = 16
RHS_SYM_FP32_PER_PAIR = 11  # symmetric kernel: 22 per unordered pair
HESS_FP32_PER_PAIR = 37
HESS_SYM_FP32_PER_PAIR = 26  # symmetric Hessian kernel: 52 per unordered pair


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


def traffic_json(n):
    """DRAM bytes per launch of the headline kernel from the latest committed ncu capture."""
    for name in ("r02_rhs_traffic.json", "r01_rhs_traffic.json"):
        try:
            tj = json.load(open(os.path.join(ROOT, "profiles", name)))
        except Exception:
            continue
        if tj.get("n") == n:
            return tj["dram_bytes_per_launch"], name
    return None, None


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
    n_sample-point input (the reference's exact path is serial per call).
    Returns ordered pair interactions per second."""
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
    sample = (f"{used} concurrent reference hamiltonian_gradients calls (FP64, serial per call) at "
              f"N={n_s} per step ({n_s}^2 ordered pairs each), extrapolated to N={args.n} by N^2 x "
              f"4 RHS/step (a full N={args.n} RHS takes hours on the host)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "flow steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 / value, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config4 exact RK4 N={args.n} (extrapolated by N^2 from a sample)",
                   "n": args.n, "sigma": SIGMA, "integrator": "rk4", "timesteps": T_STEPS},
        "pair_interactions_per_s": rate,
        "cpu_baseline": {"value": value, "unit": "flow steps/s", "cores": used, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "flow steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
def spawn_ranks(args) -> int:
    """--gpus N outside torchrun: re-launch this script with N ranks (one per GPU)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def microbench(lib, dev):
    out = {}
    for kind, name in ((0, "ffma"), (1, "ex2"), (2, "dfma"), (3, "ffma_reg"), (4, "ffma2")):
        v = C.c_double()
        lib.gs_microbench(dev, kind, C.byref(v))
        out[name] = v.value
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1907_04834_b200 import (BARNES_HUT, EULER, EXACT, F32, F64, RK4, Geoshoot,
                                       ShootingConfig, _lib)
    from paper_1907_04834_b200.shard import ShardedFlow
    from tests.util import smooth_momenta, tube

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")
    N = args.n
    q0, p0 = workload(N)
    gs = Geoshoot(local)
    lib = _lib.load()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def ev_pair():
        return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    # L2 is 126 MB and the records are 32 MB: flush it before every timed step
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    # ---- headline: exact all-pairs RK4 steps --------------------------------
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
            return flow.last_launches()
        l0 = drv.launches
        drv.step(1)
        return drv.launches - l0

    for _ in range(args.warmup):
        step()
    flow.sync()
    barrier()
    flow.profile(True)
    ev = [ev_pair() for _ in range(args.steps)]
    clocks = Clocks(local)
    launches = 0
    barrier()
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        ev[k][0].record(stream)
        launches += step()
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    flow.sync()  # raises NonFiniteState if the flow blew up
    ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev))
    prof = flow.profile_read()
    flow.profile(False)
    value = args.steps / (ms / 1e3)
    pairs_per_s = 4.0 * N * float(N) * args.steps / (ms / 1e3)

    # roofline of the dominant kernel (all-pairs RHS): FMA-pipe bound at 16 FP32
    # per pair; peak from a live FFMA microbenchmark
    mb = microbench(lib, local)
    k_ms = prof["kernel_ms"] / max(1, prof["kernel_launches"])
    pairs_per_launch = float(N) * shard
    achieved = pairs_per_launch / (k_ms * 1e-3) / 1e9  # Gpair/s
    # the symmetric kernel (unsharded, N >= 200k) evaluates each unordered pair
    # once for both ends: 22 FP32 per unordered pair = 11 per ordered pair
    tiles = gs.exact_pairs_plan(N, F32) if (world == 1 or (drv is not None and drv.pairs)) else 0
    fp32_pp = RHS_SYM_FP32_PER_PAIR if tiles else RHS_FP32_PER_PAIR
    peak = mb["ffma"] / fp32_pp / 1e9
    mp = peaks_json()
    nominal = 148 * 128 * float(mp.get("sm_max_mhz", 1965.0)) * 1e6 / fp32_pp / 1e9
    traffic, tsrc = traffic_json(N) if world == 1 else (None, None)
    roofline = {
        "bound": "fp32-fma-pipe", "achieved": achieved, "peak": peak, "unit": "Gpair/s",
        "frac": achieved / peak, "traffic": traffic,
        "traffic_unit": f"DRAM bytes per launch (ncu, profiles/{tsrc})" if tsrc else None,
        "peak_source": "live FFMA microbenchmark (gs_microbench kind 0): "
                       f"{mb['ffma'] / 1e12:.2f} T lane-FFMA/s / {fp32_pp:g} FP32 instructions per "
                       "ordered pair; MEASURED_PEAKS.json has no FP32 figure",
        "nominal_peak": nominal, "frac_of_nominal": achieved / nominal,
        "peak_register_operand_ffma": mb["ffma_reg"] / fp32_pp / 1e9,
        "peak_packed_ffma2": mb["ffma2"] / fp32_pp / 1e9,
        "sfu_frac": achieved * 1e9 / (2.0 if tiles else 1.0) / mb["ex2"] if mb["ex2"] else None,
        "kernel": ("k_rhs_sym_f32x2<12,256,1,128,8> (symmetric: each unordered pair once, fed to "
                   f"both ends; {tiles} tiles of 3072 points, packed FFMA2)") if tiles else
                  "k_rhs_f32x2<12,128,2,8> (packed FFMA2, source loop unrolled 8)",
        "kernel_ms_avg": k_ms,
        "kernel_share_of_step": prof["kernel_ms"] / (ms / 1) if ms else None,
        "algorithmic_per_launch": (f"{pairs_per_launch:.3e} ordered pairs = {pairs_per_launch / 2:.3e} "
                                   "unordered pairs x 22 FP32 + 1 MUFU") if tiles else
                                  f"{pairs_per_launch:.3e} ordered pairs x 16 FP32 + 1 MUFU",
        # the same time against the gather formulation's ceiling (16 FP32 per ordered pair)
        "frac_of_gather_ceiling": achieved / (mb["ffma"] / RHS_FP32_PER_PAIR / 1e9),
        "traffic_note": ("FMA-pipe bound: the algorithmic bytes are the 32-B records (32 MB at 1M); "
                         "the rest is the tile-slot partials the symmetric kernel writes by design "
                         "(T slots x N x 32 B, read once by the stage epilogue) -- "
                         f"{(traffic or 0) / (k_ms * 1e-3) / 1e9:.0f} GB/s during the kernel")
                        if tiles else None,
    }
    line = {
        "metric": METRIC, "value": value, "unit": "flow steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded uniform cube, BASELINE config 4)",
        "config": {"workload": f"config4: exact all-pairs RHS, RK4 x {T_STEPS} steps, N={N}, "
                               f"sigma={SIGMA}, unit cube, fp32; 1 step = 4 RHS",
                   "n": N, "sigma": SIGMA, "integrator": "rk4", "timesteps": T_STEPS,
                   "backend": "exact",
                   "parallelism": (f"pair-rows x{world} (symmetric tile-pair rows, all-to-all of "
                                   "per-target partials + all-gather of records per stage)")
                   if drv is not None and drv.pairs else f"target-shard x{world}",
                   "l2": "flushed (256 MB write) before every timed step"},
        "pair_interactions_per_s": pairs_per_s,
        "gpu_launches": launches,
        "clocks": clk,
        "roofline": roofline,
    }
    del drv, flow

    # ---- end to end through the public API, host buffers ---------------------
    pin_q = torch.empty((N, 3), dtype=torch.float64, pin_memory=True).numpy()
    pin_p = torch.empty((N, 3), dtype=torch.float64, pin_memory=True).numpy()
    pin_q[:] = q0
    pin_p[:] = p0
    if world == 1:
        t0 = time.perf_counter()
        gs.shoot_forward(pin_q, pin_p, cfg, keep_trajectory=False)
        dt = time.perf_counter() - t0
        call = f"gs_shoot_forward (10 RK4 steps, final state only) x1, {dt:.2f} s"
    else:
        fe = gs.flow(cfg, N)
        de = ShardedFlow(fe, 4)
        barrier()
        t0 = time.perf_counter()
        fe.upload(pin_q, pin_p)
        de.step(T_STEPS)
        fe.sync()
        fe.download()
        dt = max_over_ranks(time.perf_counter() - t0)
        call = (f"per rank: gs_flow_upload + {T_STEPS} sharded RK4 steps (NCCL all-gather per "
                f"stage) + gs_flow_download; max over ranks {dt:.2f} s")
        del de, fe
    line["e2e"] = {"value": T_STEPS / dt, "unit": "flow steps/s",
                   "h2d_bytes_per_step": 2 * N * 24 // T_STEPS,
                   "d2h_bytes_per_step": 2 * N * 24 // T_STEPS, "call": call}

    # ---- Barnes-Hut: exactly the config's 10 RK4 steps from q0 ----------------
    def bh_line():
        cfg_bh = ShootingConfig(sigma=SIGMA, timesteps=T_STEPS, backend=BARNES_HUT,
                                integrator=RK4, precision=F32)
        fb = gs.flow(cfg_bh, N)
        sb = torch.cuda.ExternalStream(fb.stream())

        def trajectory(timed):
            fb.upload(q0, p0)
            d = ShardedFlow(fb, 4, stream=sb) if world > 1 else None
            fb.sync()
            barrier()
            st0 = fb.stats()
            with torch.cuda.stream(sb):
                flush.zero_()
            e0, e1 = ev_pair()
            e0.record(sb)
            if d is None:
                fb.advance(T_STEPS)  # steps after the first replay a CUDA graph
            else:
                d.step(T_STEPS)
            e1.record(sb)
            torch.cuda.synchronize()
            barrier()
            fb.sync()
            return e0.elapsed_time(e1), st0, fb.stats(), (d.launches if d else fb.last_launches())

        trajectory(False)  # warm-up trajectory (allocations, graph capture)
        bms, st0, st1, bl = trajectory(True)
        bms = max_over_ranks(bms)
        d = st1["direct_interactions"] - st0["direct_interactions"]
        a_ = st1["approximated_interactions"] - st0["approximated_interactions"]
        v = st1["nodes_visited"] - st0["nodes_visited"]
        rhs = 4 * T_STEPS
        out = {"value": T_STEPS / (bms / 1e3), "unit": "flow steps/s", "ms_per_step": bms / T_STEPS,
               "timed": f"one full trajectory: {T_STEPS} RK4 steps from q0 (L2 flushed before)",
               "n2_equivalent_pairs_per_s": 4.0 * N * float(N) * T_STEPS / (bms / 1e3),
               "interactions_per_s": (d + a_) / (bms / 1e3) * world,
               "per_query_per_rhs": {"direct": d / (rhs * shard), "approximated": a_ / (rhs * shard),
                                     "visited": v / (rhs * shard)},
               "gpu_launches": bl, "parallelism": f"target-shard x{world}"}
        if world == 1:
            # per-phase kernel times: the same trajectory again, profiled (eager)
            fb.upload(q0, p0)
            fb.sync()
            fb.profile(True)
            fb.advance(T_STEPS)
            fb.sync()
            ph = fb.profile_phases(6)
            fb.profile(False)
            trav_s = ph["kernel"]["ms"] / 1e3
            build_ms = ph["build"]["ms"] / max(1, ph["build"]["count"])
            out.update({
                "traversal_ms_per_rhs": ph["kernel"]["ms"] / max(1, ph["kernel"]["count"]),
                "tree_build_ms_per_rhs": build_ms,
                "build_phases_ms_per_rhs": {k: ph[k]["ms"] / max(1, ph[k]["count"])
                                            for k in ("bbox_keys", "sort", "topology", "aggregate")},
                # 16 FP32 per interaction + 12 per visited node
                "traversal_fp32_issue_frac": ((16.0 * (d + a_) + 12.0 * v) / trav_s) / mb["ffma"]
                if trav_s > 0 else None,
                # algorithmic bytes of the build kernels, FP32 (per point)
                "build_gbs_algorithmic": BUILD_BYTES_PER_POINT * N / (build_ms * 1e-3) / 1e9,
                "build_hbm_frac": BUILD_BYTES_PER_POINT * N / (build_ms * 1e-3) / 1e9
                / float(mp.get("hbm_gbs", 6540.0)),
                "kernel": "k_bh_ws<float> (independent walks); tree: radix sort + LCP topology",
            })
        return out

    if not args.no_bh:
        try:  # an auxiliary line: never let it take the headline down
            line["bh"] = bh_line()
        except Exception as exc:  # noqa: BLE001
            line["bh"] = {"error": f"{type(exc).__name__}: {exc}"}

    # ---- exact with the FP32 underflow cutoff (opt-in), the same trajectory ----
    if not args.no_extra and world == 1:
        cfg_c = ShootingConfig(sigma=SIGMA, timesteps=T_STEPS, backend=EXACT, integrator=RK4,
                               precision=F32, exact_cutoff=True)
        fc = gs.flow(cfg_c, N)
        sc = torch.cuda.ExternalStream(fc.stream())
        fc.upload(q0, p0)
        fc.advance(T_STEPS)  # warm-up trajectory
        fc.sync()
        fc.upload(q0, p0)
        fc.sync()
        with torch.cuda.stream(sc):
            flush.zero_()
        c0, c1 = ev_pair()
        c0.record(sc)
        fc.advance(T_STEPS)
        c1.record(sc)
        torch.cuda.synchronize()
        fc.sync()
        cms = c0.elapsed_time(c1)
        line["exact_cutoff"] = {
            "value": T_STEPS / (cms / 1e3), "unit": "flow steps/s", "ms_per_step": cms / T_STEPS,
            "timed": f"one full trajectory: {T_STEPS} RK4 steps from q0",
            "speedup_vs_all_pairs": (T_STEPS / (cms / 1e3)) / value,
            "note": "exact FP32 sum in Morton order; (target group, source tile) pairs beyond "
                    "the FP32 underflow radius of 2^-r'^2 skipped (their terms are exactly 0)",
        }
        del fc

    # ---- adjoint: config 3's evaluate() (forward + kept trees + adjoint) ------
    if not args.no_extra and world == 1:
        n3 = 50_000
        q3 = tube(n3, seed=3)
        p_true = smooth_momenta(q3, 0.01, 4)  # well-conditioned amplitude
        tgt, _, _, _ = gs.shoot_forward(q3, p_true, ShootingConfig(sigma=5.0, timesteps=20),
                                        keep_trajectory=False)
        p3 = np.full_like(q3, 1e-3)
        adj = {"workload": f"config3 evaluate(): N={n3} tube, sigma 5, lambda 100, T=20 Euler, "
                           "FP32, forward flow + kept trees + adjoint, host buffers in/out"}
        for backend, name in ((EXACT, "exact"), (BARNES_HUT, "bh")):
            c3 = ShootingConfig(sigma=5.0, lambda_=100.0, timesteps=20, backend=backend, precision=F32)
            gs.evaluate(q3, p3, tgt, c3)  # warm
            gs.profile(True)
            reps = 3
            t0 = time.perf_counter()
            for _ in range(reps):
                evr = gs.evaluate(q3, p3, tgt, c3)
            dt = (time.perf_counter() - t0) / reps
            ph = gs.profile_phases()
            gs.profile(False)
            rec = {"evaluate_s": dt, "evaluations_per_s": 1.0 / dt,
                   "forward_ms": evr.stats["forward_ms"], "backward_ms": evr.stats["backward_ms"]}
            ak = ph["adjoint_kernel"]
            if backend == EXACT and ak["count"]:
                h_ms = ak["ms"] / ak["count"]
                pps = float(n3) * n3 / (h_ms * 1e-3)
                # the symmetric Hessian kernel (same size rule as the RHS) does
                # 52 FP32 per unordered pair = 26 per ordered pair
                hsym = gs.exact_pairs_plan(n3, F32) > 0
                hfp = HESS_SYM_FP32_PER_PAIR if hsym else HESS_FP32_PER_PAIR
                hpeak = mb["ffma"] / hfp
                rec["roofline"] = {
                    "bound": "fp32-fma-pipe",
                    "kernel": ("k_hess_sym_f32x2<6,128,2,64> (each unordered pair once, packed FFMA2)"
                               if hsym else "k_hess_f32x2<4,128> (packed FFMA2)"),
                    "achieved": pps / 1e9, "peak": hpeak / 1e9, "unit": "Gpair/s",
                    "frac": pps / hpeak, "kernel_ms_avg": h_ms,
                    "algorithmic_per_launch": f"{float(n3) * n3:.3e} ordered pairs x "
                                              f"{hfp} FP32 + {'1/2' if hsym else '1'} MUFU",
                    "frac_of_gather_ceiling": pps / (mb["ffma"] / HESS_FP32_PER_PAIR),
                    "peak_source": f"live FFMA microbenchmark / {hfp} FP32 per ordered pair"}
            elif ak["count"]:
                rec["adjoint_walk_ms_avg"] = ak["ms"] / ak["count"]
                rec["interactions"] = (evr.stats["direct_interactions"]
                                       + evr.stats["approximated_interactions"])
            adj[name] = rec
        line["adjoint"] = adj

    # ---- exact FP64 at N = 1M (one RK4 step) and N = 100k FP32 ----------------
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
            t0_, t1_ = ev_pair()
            t0_.record(s_)
            fl.advance(steps)
            t1_.record(s_)
            torch.cuda.synchronize()
            fl.sync()
            pr = fl.profile_read()
            fl.profile(False)
            return t0_.elapsed_time(t1_), pr
        ms64, pr64 = timed_flow(N, F64, RK4, 1)
        k64 = pr64["kernel_ms"] / max(1, pr64["kernel_launches"])
        pps64 = float(N) * N / (k64 * 1e-3)
        # DP operations per ordered pair incl. the 10-DP table-driven exp
        # (csrc/gs_exp.cuh): gather 26; symmetric 35 per unordered pair
        sym64 = gs.exact_pairs_plan(N, F64) > 0
        dp_pp = 17.5 if sym64 else 26.0
        line["fp64"] = {
            "workload": f"exact FP64, N={N}, one RK4 step (4 RHS), config-4 distribution",
            "value": 1.0 / (ms64 / 1e3), "unit": "flow steps/s", "pair_interactions_per_s": pps64,
            "kernel": ("k_rhs_sym_f64<4,256,1,64> + k_fold_group (each unordered pair once; "
                       "1024-point tiles, diagonals in groups of 32)") if sym64 else "k_rhs_f64<4,128>",
            "kernel_ms": k64, "peak_dfma_lane_per_s": mb["dfma"],
            "dp_ops_per_ordered_pair": dp_pp,
            "frac_of_dfma_peak": pps64 * dp_pp / mb["dfma"] if mb["dfma"] else None,
        }
        ms1, pr1 = timed_flow(100_000, F32, RK4, 3)
        line["n100k"] = {
            "value": 3 / (ms1 / 1e3), "unit": "flow steps/s (RK4)",
            "pair_interactions_per_s": 4.0 * 1e10 * 3 / (ms1 / 1e3),
            "frac_of_ffma_peak": (4.0 * 1e10 * 3 / (ms1 / 1e3)) / peak / 1e9,
            "kernel": ("k_rhs_sym_f32x2<12,128,2,256,4> (symmetric, 1536-point tiles)"
                       if gs.exact_pairs_plan(100_000, F32) else "k_rhs_f32x2 (gather)"),
        }

    # ---- CPU baseline: the reference's own exact RHS on the host cores ---------
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        rate, used, kind = cpu_reference(args.cpu_sample, threads)
        line["cpu_baseline"] = {
            "value": rate / (4.0 * float(N) ** 2), "unit": "flow steps/s", "cores": used,
            "kind": kind, "pair_interactions_per_s": rate,
            "sample": f"{used} concurrent reference hamiltonian_gradients calls at N={args.cpu_sample} "
                      f"(FP64, serial by construction per call), extrapolated to N={N} by N^2 x 4 RHS/step"}
        if "fp64" in line:
            line["fp64"]["vs_cpu_baseline_fp64"] = line["fp64"]["pair_interactions_per_s"] / rate
        if "bh" in line and "error" not in line["bh"] and kind == "reference":
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
    ap.add_argument("--cpu-sample", type=int, default=20_000)
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the cutoff / adjoint / FP64 / N=100k lines")
    ap.add_argument("--no-bh", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
