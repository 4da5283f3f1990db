#!/usr/bin/env python
"""bench.py -- headline benchmark: fp64 log I_v / log K_v evaluations per second.

Workload (BASELINE.json configs[1] + configs[2]): per GPU, the paper's SciPy
comparison grid -- v in {2^0..2^10}, 20M x per v uniform in [1, 100]
(220M pairs, Fig. 1 caption).  One step = log I_v(x) and log K_v(x)
of every pair (440M evaluations) in one fused pass, b200_log_ivkv_f64; the
same work as two calls (b200_log_iv_f64 then b200_log_kv_f64) is timed beside
it and reported as "separate_calls".  Inputs (3.5 GB) and outputs (3.5 GB)
live in HBM, far larger than L2.

Multi-GPU: one process per GPU.  `--gpus N` without torchrun re-launches the
command under torch.distributed.run (N ranks); under torchrun WORLD_SIZE must
equal N.  Every rank evaluates its own 220M-pair batch (weak scaling, no
data-path collective); time = max over ranks.  extra.bench_grid_strong splits
ONE 220M-pair grid contiguously over the ranks (strong scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the oracle (oracle/, binary128 CPU) on bounded samples
of the same workload -- the only reference this paper-only task has.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "logIv/logKv Gevals/s fp64"
UNIT = "Gevals/s"
N_PER_V = 20_000_000
N_ORDERS = 11
BYTES_PER_PAIR = 32          # read v, x (2 x 8 B), write log I, log K (2 x 8 B)  -- DESIGN.md §6
# FP64 operations (DADD + DMUL + 2*DFMA, thread level) and DRAM bytes per
# evaluation of the dominant kernel, from the ncu --set full capture of the
# bench workload promoted to profiles/roofline_counts.json
# (tools/summarize_profiles.py --promote).


def _roofline_counts():
    p = os.path.join(ROOT, "profiles", "roofline_counts.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _dist():
    import torch
    import torch.distributed as dist
    ws, lrank = _env_int("WORLD_SIZE", 1), _env_int("LOCAL_RANK", 0)
    if ws > 1 and not dist.is_initialized():
        torch.cuda.set_device(lrank)          # one GPU per rank before NCCL binds a device
        dist.init_process_group("nccl", device_id=torch.device("cuda", lrank))
    return ws, _env_int("RANK", 0), lrank


class Clocks:
    """SM clock / throttle-reason sampler for the timed region (B200_PROFILING.md
    clocks line): NVML every 10 ms in a thread (nvidia-smi's 200 ms floor would
    see only a couple of samples of a ~100 ms region)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        import threading
        self.sm, self.smax, self.reasons = [], 0, set()
        self.stop_ev = threading.Event()
        self.th = None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self.stop_ev.is_set():
                    try:
                        self.sm.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for nm, bit in self.REASONS.items():
                            if r & bit:
                                self.reasons.add(nm)
                    except Exception:
                        pass
                    self.stop_ev.wait(0.01)
            self.th = threading.Thread(target=run, daemon=True)
            self.th.start()
        except Exception:
            self.th = None

    def stop(self):
        if self.th is None:
            return None
        self.stop_ev.set()
        self.th.join(timeout=2)
        if not self.sm:
            return None
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.smax, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "sampler": "NVML, 10 ms"}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


def _fp64_peak():
    p = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("fp64_tflops"), d.get("source", "measured")
    return None, None


def _fp64_theoretical():
    """148 SMs x 64 FP64 FMA lanes/clk x 2 flop x the max SM clock (profiles/fp64_peak.json)."""
    p = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(p):
        return json.load(open(p)).get("theoretical_tflops_at_max_clock")
    return None


def _fn_roofline(name, evals, ms):
    """FP64 roofline of one single-function launch (flop per evaluation: ncu, profiles/roofline_counts.json)."""
    cnt = _roofline_counts().get(name, {})
    peak, src = _fp64_peak()
    fl = cnt.get("fp64_flop_per_eval")
    if not fl or not peak or ms <= 0:
        return None
    tf = fl * evals / (ms / 1e3) / 1e12
    hbm_peak, _ = _peaks()
    gbs = 24 * evals / (ms / 1e3) / 1e9
    theo = _fp64_theoretical()
    return {"bound": "alu", "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
            "frac_vs_theoretical": (tf / theo) if theo else None, "fp64_flop_per_eval": fl,
            "flop_source": cnt.get("source"), "hbm": {"achieved_gbs": gbs, "frac": gbs / hbm_peak,
                                                      "algorithmic_bytes_per_eval": 24}}


def cpu_baseline(target_s=12.0, seed=123):
    """The oracle (as it stands) on host cores, bounded sample of the same workload."""
    import numpy as np

    import oracle
    from paper_2409_08729_b200 import workloads
    cores = os.cpu_count() or 1
    n = 2000
    done_evals, done_t = 0, 0.0
    while True:
        v, x = workloads.bench_grid_numpy(max(1, n // N_ORDERS), seed=seed + n)
        t0 = time.perf_counter()
        oracle.log_iv(v, x)
        oracle.log_kv(v, x)
        dt = time.perf_counter() - t0
        done_evals += 2 * v.size
        done_t += dt
        if done_t >= target_s or n >= 50_000_000:
            break
        n = int(n * min(8.0, max(1.5, target_s / max(dt, 1e-3))))
    return {"value": done_evals / done_t / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{done_evals} evaluations (log I and log K on pairs drawn from the bench grid, "
                      f"v-major, 11 orders), binary128 oracle, OpenMP over {cores} threads, {done_t:.1f} s"}


def bench_config(n_per_v, ws):
    """The bench workload's `config` (shared by both arms: the reference arm times bounded
    samples of this same workload, described in its cpu_baseline.sample)."""
    n = N_ORDERS * n_per_v
    return {"workload": f"log I_v and log K_v of every pair of v in {{2^0..2^10}} x {n_per_v} "
                        f"x~U[1,100] per GPU ({n} pairs, v-major; configs[1]+configs[2]), "
                        "one fused pass (b200_log_ivkv_f64)",
            "pairs_per_gpu": n, "evals_per_step": 2 * n * ws,
            "l2": "inputs_larger_than_l2 (3.5 GB in, 3.5 GB out per step)",
            "parallelism": f"dp{ws} (contiguous batch per rank, no collective)"}


def run_reference(args):
    ws, rank, _ = _env_int("WORLD_SIZE", 1), _env_int("RANK", 0), 0
    if rank != 0:
        return
    import oracle
    from paper_2409_08729_b200 import workloads
    cores = os.cpu_count() or 1
    per_step = 20_000 * max(1, cores // 8)
    ts = []
    for s in range(args.warmup + args.steps):
        v, x = workloads.bench_grid_numpy(max(1, per_step // (2 * N_ORDERS)), seed=1000 + s)
        t0 = time.perf_counter()
        oracle.log_iv(v, x)
        oracle.log_kv(v, x)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            ts.append((2 * v.size, dt))
    ev = sum(e for e, _ in ts)
    tt = sum(t for _, t in ts)
    val = ev / tt / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tt / len(ts),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f128",
            "data": "synthetic",
            "config": bench_config(args.n_per_v, ws),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"each step: {ev // len(ts)} evaluations (log I and log K) on pairs "
                                       "drawn from this workload (bench grid, v-major, 11 orders), binary128, "
                                       f"OpenMP x{cores}"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _timed(step, steps, stream, dist):
    """CUDA-event time of `steps` calls of step() on `stream`, bracketed by a barrier and a
    device synchronize on both sides; max over ranks."""
    import torch
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = t0.elapsed_time(t1)
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=torch.device("cuda", torch.cuda.current_device()))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def run_extra(args, B, workloads, ws, rank, dev, stream, dist):
    """Secondary measurements on the other BASELINE configs (not the headline):
    configs[3] stability sweep (rows sharded over the ranks, strong scaling) and
    configs[4] vMF fit on 50000 x d unit-norm features (rows sharded, one
    all-reduce of the d-vector)."""
    import torch
    from paper_2409_08729_b200.parallel import shard_range
    out = {}
    # -- strong scaling of the headline: ONE global bench grid (11 x n_per_v pairs) split
    #    contiguously over the ranks (parallel.shard_range), no collective on the data path
    ntot = N_ORDERS * args.n_per_v
    g0, g1 = shard_range(ntot, ws, rank)
    gv, gx = workloads.bench_grid_slice(args.n_per_v, g0, g1, seed=0, device=dev)
    gi, gk = torch.empty_like(gv), torch.empty_like(gv)
    B.log_ivkv(gv, gx, gi, gk)
    reps = 3
    ms = _timed(lambda: B.log_ivkv(gv, gx, gi, gk), reps, stream, dist)
    out["bench_grid_strong"] = {
        "config": f"one global bench grid of {ntot} pairs (v in {{2^0..2^10}} x {args.n_per_v} x~U[1,100]) "
                  f"split contiguously over {ws} GPU(s): rank {rank} holds [{g0}, {g1})",
        "value": 2 * ntot * reps / (ms / 1e3) / 1e9, "unit": UNIT, "ms_per_step": ms / reps,
        "scaling": "strong", "time": "CUDA events, max over ranks"}
    del gv, gx, gi, gk
    # -- configs[3]: v in {0} U logspace(1e-3,1e5) x x in logspace(1e-3,1e5), 16384^2 pairs
    nv = nx = 16384
    r0, r1 = shard_range(nv, ws, rank)
    sv, sx = workloads.stability_grid(nv, nx, device=dev, rows=(r0, r1))
    oi, ok = torch.empty_like(sv), torch.empty_like(sv)
    B.log_ivkv(sv, sx, oi, ok)
    torch.cuda.synchronize()
    bad = int((~torch.isfinite(oi)).sum().item() + (~torch.isfinite(ok)).sum().item())
    if dist:
        t = torch.tensor([bad], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        bad = int(t.item())
    reps = 3
    ms = _timed(lambda: B.log_ivkv(sv, sx, oi, ok), reps, stream, dist)
    out["stability_sweep"] = {
        "config": "BASELINE configs[3]: v in {0} U logspace(1e-3,1e5) x x in logspace(1e-3,1e5), "
                  f"{nv}x{nx} = {nv * nx} pairs, rows sharded over {ws} GPU(s), fused log I + log K",
        "value": 2 * nv * nx * reps / (ms / 1e3) / 1e9, "unit": UNIT, "ms_per_pass": ms / reps,
        "nonfinite_outputs": bad, "scaling": "strong"}
    del sv, sx, oi, ok
    # -- configs[2] fp32 variant: the bench grid in float32, fused pass
    v32, x32 = workloads.bench_grid(args.n_per_v, seed=rank, device=dev, dtype=torch.float32)
    o1, o2 = torch.empty_like(v32), torch.empty_like(v32)
    B.log_ivkv(v32, x32, o1, o2)
    ms = _timed(lambda: B.log_ivkv(v32, x32, o1, o2), 3, stream, dist)
    hbm_peak, _ = _peaks()
    gbs32 = 16 * v32.numel() / (ms / 3 / 1e3) / 1e9
    out["fp32_fused"] = {"config": "configs[2] fp32 variant: bench grid in float32, b200_log_ivkv_f32",
                         "value": 2 * v32.numel() * ws * 3 / (ms / 1e3) / 1e9, "unit": UNIT,
                         "ms_per_step": ms / 3, "dtype": "f32",
                         "roofline": {"bound": "hbm", "achieved": gbs32, "peak": hbm_peak, "unit": "GB/s",
                                      "frac": gbs32 / hbm_peak, "algorithmic_bytes_per_pair": 16,
                                      "floor_ms": 16 * v32.numel() / (hbm_peak * 1e9) * 1e3,
                                      "note": "16 B per pair (v, x in; log I, log K out, float32); the f32 "
                                              "kernel is issue-bound, so this is the distance to the HBM floor"}}
    del v32, x32, o1, o2
    # -- the paper's own runtime table (Table 5): 10M fractional-order
    #    pairs uniform on the Small [0,150]^2 / Large [150,1e4]^2 (I) or [150,4000]^2 (K)
    #    regions, each function timed alone.  Context only (RTX 2080 Ti there, B200 here).
    paper_ms = {("log_iv", "small"): 50.41, ("log_iv", "large"): 39.68,
                ("log_kv", "small"): 430.60, ("log_kv", "large"): 39.96}
    pr = {}
    for (fn, region), pms in paper_ms.items():
        vv, xx = workloads.paper_region(10_000_000, region, "iv" if fn == "log_iv" else "kv", seed=7)
        vt = torch.tensor(vv, device=dev)
        xt = torch.tensor(xx, device=dev)
        ot = torch.empty_like(vt)
        f = getattr(B, fn)
        f(vt, xt, out=ot)
        ms = _timed(lambda: f(vt, xt, out=ot), 5, stream, None) / 5
        pr[f"{fn}/{region}"] = {"ms_per_10M": ms, "paper_rtx2080ti_ms_per_10M": pms,
                                "ratio_vs_paper_gpu": pms / ms}
        del vt, xt, ot
    out["paper_table5_context"] = {
        "note": "PAPER.md Table 5 (CUSF GPU column, RTX 2080 Ti, fp64, 10M pairs per region): another "
                "machine's numbers, quoted as context, not as the target; the paper's abstract reports "
                "median/max GPU speedups of 45x/6150x over third-party libraries and 77x/300x over SciPy",
        "regions": pr}
    # -- configs[4]: vMF MLE on 50000 x d features (f32), rows sharded
    n = 50_000
    lo, hi = shard_range(n, ws, rank)
    hbm_peak, _ = _peaks()
    vm = {}
    for d in (2048, 8192, 32768):
        # rows [lo, hi) of ONE 50000 x d matrix (mu and every row independent of the world size)
        X, _ = workloads.vmf_features(n, d, rbar=0.15, seed=100, device=dev, rows=(lo, hi))
        pg = dist.group.WORLD if dist else None
        mu, st = B.vmf_fit(X, process_group=pg)
        torch.cuda.synchronize()
        reps = 5
        ms = _timed(lambda: B.vmf_fit(X, process_group=pg), reps, stream, dist)
        cs = torch.empty(d + 1, dtype=torch.float64, device=dev)
        ms_cs = _timed(lambda: B.vmf_colsum(X, out=cs, with_count=True), reps, stream, None)
        gbs = (hi - lo) * d * 4 / (ms_cs / reps / 1e3) / 1e9
        vm[str(d)] = {"ms_per_fit": ms / reps, "colsum_ms": ms_cs / reps,
                      "colsum_roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
                                          "frac": gbs / hbm_peak},
                      "rbar": float(st[0].item()), "kappa_mle": float(st[4].item())}
        del X
    out["vmf_fit"] = {"config": f"BASELINE configs[4]: one {n} x d unit-norm f32 feature matrix (Rbar 0.15), "
                                f"rows sharded over {ws} GPU(s), one all-reduce of d + 1 doubles (column sums "
                                "and the row count)", "per_d": vm}
    return out


def run_ours(args):
    import torch

    import paper_2409_08729_b200 as B
    from paper_2409_08729_b200 import workloads
    ws, rank, lrank = _dist()
    torch.cuda.set_device(lrank)
    dev = torch.device("cuda", lrank)
    dist = None
    if ws > 1:
        import torch.distributed as dist

    n_per_v = args.n_per_v
    v, x = workloads.bench_grid(n_per_v, seed=rank, device=dev)
    n = v.numel()
    out_i = torch.empty_like(v)
    out_k = torch.empty_like(v)
    stream = torch.cuda.current_stream(dev)
    evals_per_step = 2 * n * ws

    # ---- the step: log I_v(x) and log K_v(x) of every pair, one fused pass (b200_log_ivkv_f64)
    def step():
        B.log_ivkv(v, x, out_i, out_k)

    # clock sampler from the warm-up through the timed region (NVML needs a few ms to start)
    clocks = Clocks(lrank) if rank == 0 else None
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # non-finite guard on the warm-up outputs (the method never produces inf/NaN here)
    nonfinite = int((~torch.isfinite(out_i)).sum().item() + (~torch.isfinite(out_k)).sum().item())
    launches0 = B.launch_count()
    ms = _timed(step, args.steps, stream, dist)
    launches = B.launch_count() - launches0
    clk = clocks.stop() if clocks else None
    value = evals_per_step * args.steps / (ms / 1e3) / 1e9

    # ---- the same work as two separate calls (b200_log_iv_f64, then b200_log_kv_f64)
    sep = None
    if not args.skip_separate:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        acc = [0.0, 0.0]

        def step_sep():
            ev[0].record(stream)
            B.log_iv(v, x, out=out_i)
            ev[1].record(stream)
            B.log_kv(v, x, out=out_k)
            ev[2].record(stream)

        def step_sep_acc():
            step_sep()
            torch.cuda.synchronize()
            acc[0] += ev[0].elapsed_time(ev[1])
            acc[1] += ev[1].elapsed_time(ev[2])
        for _ in range(args.warmup):
            step_sep()
        ms_sep = _timed(step_sep, args.steps, stream, dist)
        for _ in range(args.steps):
            step_sep_acc()
        kiv, kkv = acc[0] / args.steps, acc[1] / args.steps
        sep = {"value": evals_per_step * args.steps / (ms_sep / 1e3) / 1e9, "unit": UNIT,
               "ms_per_step": ms_sep / args.steps,
               "kernel_ms": {"log_iv": kiv, "log_kv": kkv},
               "roofline": {"log_iv": _fn_roofline("log_iv", n, kiv), "log_kv": _fn_roofline("log_kv", n, kkv)},
               "note": "b200_log_iv_f64 then b200_log_kv_f64 over the same grid (2 launches per step); "
                       "per-function FP64 roofline from CUDA events around each launch"}

    # ---- end to end through the C ABI with pinned HOST buffers (H2D + kernel + D2H timed)
    e2e = None
    if not args.skip_e2e:
        # the first E2E_PAIRS pairs of this rank's grid (all 11 orders at full size is
        # 7 GB of pinned host memory per rank; the metric is a rate)
        ne = min(n, args.e2e_pairs)
        sel = torch.arange(ne, device=dev) * (n // ne) if ne < n else slice(None)
        vh = v[sel].cpu().pin_memory()
        xh = x[sel].cpu().pin_memory()
        oi = torch.empty_like(vh, pin_memory=True)
        ok = torch.empty_like(vh, pin_memory=True)
        B.log_ivkv_host(vh, xh, oi, ok)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        reps = max(1, min(args.steps, 3))
        for _ in range(reps):
            B.log_ivkv_host(vh, xh, oi, ok)
        te = time.perf_counter() - t0
        if dist:
            t = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": 2 * ne * ws * reps / te / 1e9, "unit": UNIT,
               "pairs_per_step": ne * ws,
               "h2d_bytes_per_step": 2 * ne * 8 * ws, "d2h_bytes_per_step": 2 * ne * 8 * ws,
               "note": "b200_log_ivkv_f64_host on pinned host arrays (every (n/e2e_pairs)-th pair of the "
                       "bench grid, all orders): v, x cross PCIe once per pair, both results come back; "
                       "chunked H2D/kernel/D2H pipeline on 4 streams (4M-pair chunks); host wall clock, max over ranks; "
                       "bytes and pairs are whole-job"}
        del vh, xh, oi, ok

    extra = None if args.skip_extra else run_extra(args, B, workloads, ws, rank, dev, stream, dist)
    del v, x, out_i, out_k
    if rank != 0:
        return
    hbm_peak, hbm_src = _peaks()
    kms = ms / args.steps                      # one launch per step: the step is the kernel
    gbs = BYTES_PER_PAIR * n / (kms / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
            "traffic": None, "kernel": "bessel_eval_kernel<double, FN_IK> (b200_log_ivkv_f64)",
            "peak_source": hbm_src, "kernel_ms": kms}
    fp64_peak, fp64_src = _fp64_peak()
    cnt = _roofline_counts().get("log_ivkv", {})
    fl = cnt.get("fp64_flop_per_eval")         # per pair (two evaluations)
    if cnt.get("dram_bytes_per_eval"):
        roof["traffic"] = cnt["dram_bytes_per_eval"] * n          # bytes per launch of this step
        roof["traffic_source"] = (cnt["source"] + f"; dram read+write {cnt['dram_bytes_per_eval']:.2f} B per pair "
                                  f"(ncu) x {n} pairs; algorithmic {BYTES_PER_PAIR} B per pair")
    if fl and fp64_peak:
        tf = fl * n / (kms / 1e3) / 1e12
        if tf / fp64_peak > gbs / hbm_peak:
            roof = {"bound": "alu", "achieved": tf, "peak": fp64_peak, "unit": "TFLOP/s",
                    "frac": tf / fp64_peak, "traffic": roof.get("traffic"),
                    "traffic_source": roof.get("traffic_source"),
                    "kernel": "bessel_eval_kernel<double, FN_IK> (b200_log_ivkv_f64)",
                    "peak_source": fp64_src, "kernel_ms": kms, "fp64_flop_per_pair": fl,
                    "flop_source": cnt["source"] + " (DADD + DMUL + 2 DFMA executed per pair)",
                    "hbm": {"achieved_gbs": gbs, "peak_gbs": hbm_peak, "frac": gbs / hbm_peak,
                            "algorithmic_bytes_per_pair": BYTES_PER_PAIR}}
            theo = _fp64_theoretical()
            if theo:
                roof["frac_vs_theoretical"] = tf / theo
                roof["theoretical_peak"] = theo
            fi = cnt.get("fp64_inst_per_eval")
            if fi:
                # FP64-pipe occupancy view: a DADD or DMUL takes a pipe slot like a DFMA
                # but counts one flop, so the flop fraction understates pipe use
                ti = fi * n / (kms / 1e3) / 1e12
                roof["fp64_pipe"] = {"achieved_tinst_s": ti, "peak_tinst_s": fp64_peak / 2,
                                     "frac": ti / (fp64_peak / 2), "fp64_inst_per_pair": fi,
                                     "note": "DADD + DMUL + DFMA issued per pair (ncu) x pairs/s vs the "
                                             "measured DFMA issue rate (peak FLOP/s / 2)"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(n_per_v, ws),
        "roofline": roof,
        "gpu_launches": launches,
        "nonfinite_outputs": nonfinite,
        "separate_calls": sep,
        "extra": extra,
        "e2e": e2e,
        "clocks": clk,
    }
    if not args.skip_cpu_baseline and ws == 1:
        line["cpu_baseline"] = cpu_baseline(args.cpu_seconds)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n-per-v", type=int, default=N_PER_V)
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-separate", action="store_true")
    ap.add_argument("--skip-extra", action="store_true")
    ap.add_argument("--e2e-pairs", type=int, default=55_000_000,
                    help="pairs per rank in the end-to-end (host buffer) measurement")
    ap.add_argument("--skip-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None and args.gpus > 1:
        # one process per GPU: re-launch this command under torch.distributed.run
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)
    if ws_env is not None and int(ws_env) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env} (launch one process per GPU, "
              "or omit torchrun and let --gpus spawn them)", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
    try:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()
    except Exception:
        pass


if __name__ == "__main__":
    main()
