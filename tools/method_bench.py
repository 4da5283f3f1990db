"""Per-slice / per-method timing of the evaluation kernels (diagnostic; not the bench).

For each order v of the bench grid (20M x ~ U[1,100]) and for method-homogeneous
input sets, time b200_log_iv_f64 / b200_log_kv_f64 with CUDA events.
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2409_08729_b200 as B  # noqa: E402


def timeit(f, v, x, reps=5):
    out = torch.empty_like(v)
    f(v, x, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f(v, x, out=out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    dev = torch.device("cuda:0")
    n = 20_000_000
    g = torch.Generator(device=dev).manual_seed(0)
    res = {"per_v": {}, "per_method": {}}
    x = torch.empty(n, dtype=torch.float64, device=dev).uniform_(1.0, 100.0, generator=g)
    for j in range(11):
        v = torch.full((n,), float(2 ** j), dtype=torch.float64, device=dev)
        res["per_v"][str(2 ** j)] = {fn: timeit(getattr(B, fn), v, x) for fn in ("log_iv", "log_kv")}
    sets = {
        "mu": ((0.0, 15.0), (30.0, 100.0)),
        "u4": ((2000.0, 2000.0), (1.0, 100.0)),
        "u6": ((512.0, 1024.0), (1.0, 100.0)),
        "u9": ((100.0, 256.0), (1.0, 60.0)),
        "u13": ((13.0, 60.0), (1.0, 40.0)),
        "fallback_a": ((0.8, 12.0), (0.3, 2.0)),
        "fallback_b": ((0.8, 12.0), (8.1, 19.0)),
    }
    for name, ((v0, v1), (x0, x1)) in sets.items():
        v = torch.empty(n, dtype=torch.float64, device=dev).uniform_(v0, v1, generator=g)
        xx = torch.empty(n, dtype=torch.float64, device=dev).uniform_(x0, x1, generator=g)
        res["per_method"][name] = {fn: timeit(getattr(B, fn), v, xx) for fn in ("log_iv", "log_kv")}
    for k in res:
        for kk, d in res[k].items():
            d.update({f"{fn}_gevals": n / (ms * 1e-3) / 1e9 for fn, ms in list(d.items())})
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
