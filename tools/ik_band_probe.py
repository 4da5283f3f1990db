"""Fused-pass fallback probe: time and accuracy of build/variants/<name>.so builds
(tools/variant_bench.py build ...) on the bands where the fused pass takes
log I from the K values.  Diagnostic tool, not the bench; GPU.

  python tools/ik_band_probe.py NAME ...

Per variant: f32 fused bench grid (11 x 20M pairs), f64 fused stability sweep
(BASELINE configs[3] axes, 16384 x 16384 pairs), and max rel_err (R1)
against the oracle of both fused outputs on the 2 < x <= 30 band and the
x <= 2 band (v <= 12.69), in f64 and f32.
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import oracle  # noqa: E402
from paper_2409_08729_b200 import workloads  # noqa: E402

dev = torch.device("cuda:0")


def timed(f, args, reps=5):
    f(*args)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f(*args)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main(names):
    n = 20_000_000
    g = torch.Generator(device=dev).manual_seed(0)
    x32 = torch.empty(n, dtype=torch.float32, device=dev).uniform_(1.0, 100.0, generator=g)
    va, xa = workloads.stability_axes()
    vs = torch.tensor(va, device=dev).repeat_interleave(xa.size)
    xs = torch.tensor(xa, device=dev).repeat(va.size)
    rng = np.random.default_rng(5)
    bands = {"trap": (rng.uniform(0, 12.69, 20000), rng.uniform(2.0, 30.0, 20000)),
             "temme": (rng.uniform(0, 12.69, 20000), workloads.log_uniform(20000, 1e-8, 2.0, seed=6))}
    refs = {b: (oracle.log_iv(v, x), oracle.log_kv(v, x)) for b, (v, x) in bands.items()}
    refs32 = {b: (oracle.log_iv(v.astype(np.float32).astype(np.float64), x.astype(np.float32).astype(np.float64)),
                  oracle.log_kv(v.astype(np.float32).astype(np.float64), x.astype(np.float32).astype(np.float64)))
              for b, (v, x) in bands.items()}
    s = torch.cuda.current_stream().cuda_stream
    res = {}
    for nm in names:
        L = ctypes.CDLL(f"build/variants/{nm}.so")
        f32, f64 = L.b200_log_ivkv_f32, L.b200_log_ivkv_f64
        for f in (f32, f64):
            f.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_void_p]
        row = {}
        tot = 0.0
        for j in range(11):
            v = torch.full((n,), float(2 ** j), dtype=torch.float32, device=dev)
            o1, o2 = torch.empty_like(v), torch.empty_like(v)
            tot += timed(f32, (v.data_ptr(), x32.data_ptr(), o1.data_ptr(), o2.data_ptr(), n, s))
        row["bench_grid_f32_ms"] = round(tot, 4)
        o1, o2 = torch.empty_like(vs), torch.empty_like(vs)
        row["sweep_f64_ms"] = round(timed(f64, (vs.data_ptr(), xs.data_ptr(), o1.data_ptr(), o2.data_ptr(),
                                                vs.numel(), s), reps=3), 4)
        del o1, o2
        for b, (v, x) in bands.items():
            for dt, f, ref in ((torch.float64, f64, refs[b]), (torch.float32, f32, refs32[b])):
                vt, xt = torch.tensor(v, device=dev, dtype=dt), torch.tensor(x, device=dev, dtype=dt)
                a, c = torch.empty_like(vt), torch.empty_like(vt)
                f(vt.data_ptr(), xt.data_ptr(), a.data_ptr(), c.data_ptr(), v.size, s)
                torch.cuda.synchronize()
                key = f"{b}_{'f64' if dt == torch.float64 else 'f32'}"
                row[key] = {"err_i": float(oracle.rel_err(a.double().cpu().numpy(), ref[0]).max()),
                            "err_k": float(oracle.rel_err(c.double().cpu().numpy(), ref[1]).max())}
        res[nm] = row
        print(nm, json.dumps(row), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main(sys.argv[1:])
