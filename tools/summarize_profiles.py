#!/usr/bin/env python
"""Turn one gpurun_out/<tag>/ directory into the committed profiles/<tag>/ summaries.

  python tools/summarize_profiles.py <tag> [--pairs N]

Writes
  profiles/<tag>/launches.txt     per-kernel launch list (ncu gpu__time_duration, cold, serialised)
  profiles/<tag>/ncu_full.json    per-kernel counters of the `ncu --set full` capture
  profiles/<tag>/ncu_sass.txt     opcode mix / stall reasons / hottest SASS (tools/ncu_sass_hotspots.py)
  profiles/<tag>/bench.json       the bench line of that session (copied)
and copies fp64_peak.json to profiles/fp64_peak.json (read by bench.py).

--pairs is the number of (v, x) pairs per launch in the full capture
(bench.py --n-per-v 2000000 => 22M) and turns counts into per-evaluation figures.
"""
import collections
import csv
import json
import re
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(src, dst):
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    h = rows[0]
    agg = collections.OrderedDict()
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"]
        k = k[:k.find("(")] if "(" in k else k
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1e-3)
        agg.setdefault(k, []).append(float(d["Metric Value"]) * scale)
    tot = sum(sum(v) for v in agg.values())
    ours = sum(sum(v) for k, v in agg.items() if "b200::" in k)
    with open(dst, "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
        f.write("# kernel | launches | mean us | share of all device time\n")
        for k, v in agg.items():
            f.write(f"{k[:90]:90s} {len(v):4d} {sum(v) / len(v):12.1f} {100 * sum(v) / tot:6.2f}%\n")
        f.write(f"# b200:: kernels: {100 * ours / tot:.2f}% of device time in this process "
                "(the rest is input generation outside the timed region)\n")


def full(rep, dst, pairs):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))

        def g(k, default=None):
            try:
                return float(d[k])
            except (KeyError, ValueError):
                return default
        cyc = g("smsp__cycles_elapsed.avg")
        ops = {}
        for op in ("dadd", "dmul", "dfma"):
            rate = g(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed")
            ops[op] = rate * cyc if rate is not None and cyc else None
        flops = ops["dadd"] + ops["dmul"] + 2 * ops["dfma"] if all(ops.values()) else None
        dur_us = g("gpu__time_duration.sum")
        e = {
            "kernel": d["Kernel Name"],
            "duration_us": dur_us,
            "dram_bytes_read": g("dram__bytes_read.sum"),
            "dram_bytes_write": g("dram__bytes_write.sum"),
            "dram_unit": "MB" ,
            "registers": g("launch__registers_per_thread"),
            "fp64_pipe_active_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": g("sm__inst_issued.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "inst_executed": g("smsp__inst_executed.sum"),
            "fp64_thread_ops": ops,
            "fp64_flops": flops,
        }
        if pairs:
            e["pairs"] = pairs
            if flops:
                e["fp64_flop_per_eval"] = flops / pairs
                e["fp64_tflops"] = flops / (dur_us * 1e-6) / 1e12
            for k in ("dadd", "dmul", "dfma"):
                if ops[k]:
                    e[f"{k}_per_eval"] = ops[k] / pairs
            if e["dram_bytes_read"] is not None:
                e["dram_bytes_per_eval"] = (e["dram_bytes_read"] + e["dram_bytes_write"]) * 1e6 / pairs
        res.append(e)
    json.dump(res, open(dst, "w"), indent=1)
    return res


def main():
    tag = sys.argv[1]
    pairs = int(sys.argv[sys.argv.index("--pairs") + 1]) if "--pairs" in sys.argv else 22_000_000
    src = os.path.join(ROOT, "gpurun_out", tag)
    dst = os.path.join(ROOT, "profiles", tag)
    os.makedirs(dst, exist_ok=True)
    if os.path.exists(os.path.join(src, "launches.csv")):
        launches(os.path.join(src, "launches.csv"), os.path.join(dst, "launches.txt"))
    rep = os.path.join(src, "prof.ncu-rep")
    if os.path.exists(rep):
        r = full(rep, os.path.join(dst, "ncu_full.json"), pairs)
        for e in r:
            print(e["kernel"][:60], {k: e.get(k) for k in ("duration_us", "fp64_flop_per_eval", "fp64_tflops",
                                                            "fp64_pipe_active_pct", "dram_bytes_per_eval")})
        txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_sass_hotspots.py"), rep],
                             capture_output=True, text=True).stdout
        open(os.path.join(dst, "ncu_sass.txt"), "w").write(txt)
    for name in ("bench.json", "pytest_gpu.log", "smoke.log", "methods.json", "gpu.txt"):
        p = os.path.join(src, name)
        if os.path.exists(p):
            shutil.copy(p, os.path.join(dst, name))
    if "--promote" in sys.argv and os.path.exists(os.path.join(dst, "ncu_full.json")):
        counts = {}
        for e in json.load(open(os.path.join(dst, "ncu_full.json"))):
            m = re.search(r"bessel_eval_kernel<double, (?:\(int\))?(\d)[,>]", e["kernel"])
            fn = {"0": "log_iv", "1": "log_kv", "3": "log_ivkv"}.get(m.group(1)) if m else None
            if fn and "double" in e["kernel"] and "bessel_eval_kernel" in e["kernel"] and e.get("fp64_flop_per_eval"):
                counts[fn] = {"fp64_flop_per_eval": e["fp64_flop_per_eval"],
                              "fp64_inst_per_eval": sum(e.get(f"{k}_per_eval", 0.0) for k in ("dadd", "dmul", "dfma")),
                              "per": "pair (log I and log K)" if fn == "log_ivkv" else "evaluation",
                              "dram_bytes_per_eval": e.get("dram_bytes_per_eval"),
                              "source": f"profiles/{tag}/ncu_full.json ({e['pairs']} pairs, bench grid)"}
        json.dump(counts, open(os.path.join(ROOT, "profiles", "roofline_counts.json"), "w"), indent=1)
        print("promoted", counts)
    p = os.path.join(src, "fp64_peak.json")
    if os.path.exists(p) and os.path.getsize(p) > 0:
        shutil.copy(p, os.path.join(ROOT, "profiles", "fp64_peak.json"))


if __name__ == "__main__":
    main()
