"""Kernel design experiments: build libbessel_b200.so variants (-D macros) and time them.

Diagnostic tool, not the bench.  Each variant is the product source compiled
with extra macros into build/variants/<name>.so; every variant is timed with
CUDA events on the per-order slices of the bench grid (20M x ~ U[1,100] per v)
and on method-homogeneous input sets, and its outputs are compared with the
first variant's (max |diff| / max(|ref|,1)) as a sanity check.

  python tools/variant_bench.py build  NAME=FLAGS ...     (CPU: nvcc only)
  python tools/variant_bench.py run    NAME ...           (GPU)
FLAGS is a comma-separated list of macro definitions, e.g. B200_MINB=4,B200_EVAL_NOP.
"""
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build", "variants")


def build(specs):
    from paper_2409_08729_b200 import _build
    _build.gen_tables.write() if hasattr(_build, "gen_tables") else None
    os.makedirs(OUT, exist_ok=True)
    procs = []
    for spec in specs:
        name, _, flags = spec.partition("=")
        # items starting with '+' are raw nvcc flags ('+' stripped, '=' kept), the rest macros
        defs = [f[1:] if f.startswith("+") else f"-D{f}" for f in flags.split(",") if f]
        cmd = [_build.nvcc()] + _build.NVCC_FLAGS + defs + ["-o", os.path.join(OUT, name + ".so")] + \
              [os.path.join(_build.CSRC, s) for s in _build.SOURCES]
        procs.append((name, subprocess.Popen(cmd)))
    for name, p in procs:
        if p.wait() != 0:
            raise SystemExit(f"build of {name} failed")
        print("built", name)


def run(names, n=20_000_000, reps=5):
    import torch
    dev = torch.device("cuda:0")
    libs = {}
    for nm in names:
        L = ctypes.CDLL(os.path.join(OUT, nm + ".so"))
        for f in ("b200_log_iv_f64", "b200_log_kv_f64"):
            getattr(L, f).argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_void_p]
            getattr(L, f).restype = ctypes.c_int
        if hasattr(L, "b200_log_ivkv_f64"):
            L.b200_log_ivkv_f64.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_void_p]
            L.b200_log_ivkv_f64.restype = ctypes.c_int
        if hasattr(L, "b200_log_ivkv_f32"):
            L.b200_log_ivkv_f32.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_void_p]
            L.b200_log_ivkv_f32.restype = ctypes.c_int
        libs[nm] = L
    g = torch.Generator(device=dev).manual_seed(0)
    sets = {}
    x = torch.empty(n, dtype=torch.float64, device=dev).uniform_(1.0, 100.0, generator=g)
    for j in range(11):
        sets[f"v={2 ** j}"] = (torch.full((n,), float(2 ** j), dtype=torch.float64, device=dev), x)
    boxes = {
        "mu": ((0.0, 15.0), (30.0, 100.0)),
        "u4": ((2000.0, 2000.0), (1.0, 100.0)),
        "u6": ((512.0, 1024.0), (1.0, 100.0)),
        "u9": ((100.0, 256.0), (1.0, 60.0)),
        "u13": ((13.0, 60.0), (1.0, 40.0)),
        "fb_a": ((0.8, 12.0), (0.3, 2.0)),
        "fb_b": ((0.8, 12.0), (2.1, 19.0)),
    }
    for name, ((v0, v1), (x0, x1)) in boxes.items():
        v = torch.empty(n, dtype=torch.float64, device=dev).uniform_(v0, v1, generator=g)
        xx = torch.empty(n, dtype=torch.float64, device=dev).uniform_(x0, x1, generator=g)
        sets[name] = (v, xx)
    # divergence diagnostics: the fallback sets with the same pairs ordered by x (the trapezoid
    # node count and Miller length follow x), so every warp sees nearly equal trip counts
    for name in ("fb_a", "fb_b"):
        v, xx = sets[name]
        xs, perm = torch.sort(xx)
        sets[name + "_xsorted"] = (v[perm].contiguous(), xs.contiguous())
    s = torch.cuda.current_stream(dev).cuda_stream
    res = {}
    for sname, (v, xx) in sets.items():
        ref = {}
        for nm, L in libs.items():
            row = {}
            for fn in ("log_iv", "log_kv"):
                f = getattr(L, f"b200_{fn}_f64")
                out = torch.empty_like(v)
                f(v.data_ptr(), xx.data_ptr(), out.data_ptr(), n, s)
                torch.cuda.synchronize()
                if fn not in ref:
                    ref[fn] = out.clone()
                    dev_ = 0.0
                else:
                    dev_ = float(((out - ref[fn]).abs() / ref[fn].abs().clamp_min(1.0)).max())
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    f(v.data_ptr(), xx.data_ptr(), out.data_ptr(), n, s)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
                row[fn] = {"ms": round(ms, 4), "gevals": round(n / ms / 1e6, 2), "maxdiff": dev_}
            if hasattr(L, "b200_log_ivkv_f64"):
                o1, o2 = torch.empty_like(v), torch.empty_like(v)
                L.b200_log_ivkv_f64(v.data_ptr(), xx.data_ptr(), o1.data_ptr(), o2.data_ptr(), n, s)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    L.b200_log_ivkv_f64(v.data_ptr(), xx.data_ptr(), o1.data_ptr(), o2.data_ptr(), n, s)
                e1.record()
                torch.cuda.synchronize()
                row["ivkv"] = {"ms": round(e0.elapsed_time(e1) / reps, 4),
                               "maxdiff": max(float(((o1 - ref["log_iv"]).abs() / ref["log_iv"].abs().clamp_min(1.0)).max()),
                                              float(((o2 - ref["log_kv"]).abs() / ref["log_kv"].abs().clamp_min(1.0)).max()))}
            if hasattr(L, "b200_log_ivkv_f32"):
                v32, x32 = v.float(), xx.float()
                o1, o2 = torch.empty_like(v32), torch.empty_like(v32)
                L.b200_log_ivkv_f32(v32.data_ptr(), x32.data_ptr(), o1.data_ptr(), o2.data_ptr(), n, s)
                if "ref32" not in ref:
                    ref["ref32"] = (o1.clone(), o2.clone())
                md = max(float(((o1 - ref["ref32"][0]).abs() / ref["ref32"][0].abs().clamp_min(1.0)).max()),
                         float(((o2 - ref["ref32"][1]).abs() / ref["ref32"][1].abs().clamp_min(1.0)).max()))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    L.b200_log_ivkv_f32(v32.data_ptr(), x32.data_ptr(), o1.data_ptr(), o2.data_ptr(), n, s)
                e1.record()
                torch.cuda.synchronize()
                row["ivkv32"] = {"ms": round(e0.elapsed_time(e1) / reps, 4), "maxdiff": md}
                del v32, x32, o1, o2
            res.setdefault(sname, {})[nm] = row
    # bench-grid totals (sum over the 11 order slices)
    tot = {nm: {fn: round(sum(res[f"v={2 ** j}"][nm][fn]["ms"] for j in range(11)), 3)
                for fn in ("log_iv", "log_kv", "ivkv", "ivkv32") if fn in res["v=1"][nm]} for nm in names}
    print(json.dumps({"sets": res, "bench_grid_ms": tot}, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        run(sys.argv[2:])
