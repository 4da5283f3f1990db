"""Method-homogeneous launches for ncu (diagnostic).  Launch order: for each set in SETS,
log_iv then log_kv, n pairs each.  Parse the capture with tools/ncu_sets.py parse <rep>."""
import csv
import json
import subprocess
import sys

SETS = [
    ("mu", (0.0, 15.0), (30.0, 100.0)),
    ("u4", (2000.0, 2000.0), (1.0, 100.0)),
    ("u6", (512.0, 1024.0), (1.0, 100.0)),
    ("u9", (100.0, 256.0), (1.0, 60.0)),
    ("u13", (13.0, 60.0), (1.0, 40.0)),
    ("fb_a", (0.8, 12.0), (0.3, 2.0)),
    ("fb_b", (0.8, 12.0), (2.1, 19.0)),
    ("grid_v1", (1.0, 1.0), (1.0, 100.0)),
]


def run(n=4_000_000, fused=False, dtype="f64"):
    import torch
    sys.path.insert(0, ".")
    import paper_2409_08729_b200 as B
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    for name, (v0, v1), (x0, x1) in SETS:
        v = torch.empty(n, dtype=torch.float64, device=dev).uniform_(v0, v1, generator=g)
        x = torch.empty(n, dtype=torch.float64, device=dev).uniform_(x0, x1, generator=g)
        if dtype == "f32":
            v, x = v.float(), x.float()
        if fused:
            B.log_ivkv(v, x)
        else:
            B.log_iv(v, x)
            B.log_kv(v, x)
    torch.cuda.synchronize()


def parse(rep, n=4_000_000, fused=False):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    names = [f"{s[0]}/{fn}" for s in SETS for fn in (("IK",) if fused else ("I", "K"))]
    res = {}
    for i, r in enumerate(rows[2:]):
        d = dict(zip(h, r))

        def g(k):
            try:
                return float(d[k].replace(",", ""))
            except (KeyError, ValueError):
                return None
        cyc = g("smsp__cycles_elapsed.avg")
        ops = {op: (g(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed") or 0) * cyc
               for op in ("dadd", "dmul", "dfma")}
        stalls = {k.split("issue_stalled_")[1].split("_per_")[0]: g(k) for k in h
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")}
        top = dict(sorted(((k, round(v, 2)) for k, v in stalls.items() if v), key=lambda t: -t[1])[:6])
        res[names[i] if i < len(names) else str(i)] = {
            "us": g("gpu__time_duration.sum"),
            "inst_per_eval": 32 * g("smsp__inst_executed.sum") / n,
            "fp64_inst_per_eval": (ops["dadd"] + ops["dmul"] + ops["dfma"]) / n,
            "fp64_pipe_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_pct": g("sm__inst_issued.avg.pct_of_peak_sustained_active"),
            "warps_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "stalls_per_issue": top,
        }
    for k, v in res.items():
        print(f"{k:10s} {v['us']:8.1f}us inst/eval {v['inst_per_eval']:7.1f} fp64/eval {v['fp64_inst_per_eval']:6.1f} "
              f"fp64pipe {v['fp64_pipe_pct']:5.1f}% issue {v['issue_pct']:5.1f}% warps {v['warps_pct']:5.1f}% {v['stalls_per_issue']}")
    return res


if __name__ == "__main__":
    fz = "--fused" in sys.argv
    dt = "f32" if "--f32" in sys.argv else "f64"
    args = [a for a in sys.argv[1:] if a not in ("--fused", "--f32")]
    if args and args[0] == "parse":
        r = parse(args[1], fused=fz)
        if len(args) > 2:
            json.dump(r, open(args[2], "w"), indent=1)
    else:
        run(fused=fz, dtype=dt)
