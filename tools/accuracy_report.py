"""Max error of the CUDA path against the oracle per method-homogeneous set (diagnostic).
Run on a GPU box; prints one line per set: max rel_err (R1) of log I and log K."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2409_08729_b200 as B  # noqa: E402

SETS = {
    "mu": ((0.0, 15.0), (30.0, 100.0)), "mu_far": ((0.0, 200.0), (1e3, 1e5)),
    "u6": ((280.0, 1e5), (1.0, 1e5)), "u8": ((107.0, 277.0), (1.0, 107.0)),
    "u10": ((61.0, 107.0), (1.0, 60.0)), "u13": ((13.0, 61.0), (1.0, 60.0)),
    "u13_lowv": ((0.7, 13.0), (19.7, 30.0)), "fb_a": ((0.0, 12.69), (1e-3, 2.0)),
    "fb_b": ((0.0, 12.69), (2.0, 19.69)), "fb_b_lowv": ((0.0, 0.7), (2.0, 30.0)),
}


def main(n=20000, seed=0, dtype=torch.float64):
    rng = np.random.default_rng(seed)
    res = {}
    for name, ((v0, v1), (x0, x1)) in SETS.items():
        v = rng.uniform(v0, v1, n)
        x = np.exp(rng.uniform(np.log(x0), np.log(x1), n)) if x1 / x0 > 50 else rng.uniform(x0, x1, n)
        if dtype == torch.float32:          # the oracle at the inputs the f32 kernels see
            v = v.astype(np.float32).astype(np.float64)
            x = x.astype(np.float32).astype(np.float64)
        vt = torch.tensor(v, device="cuda:0", dtype=dtype)
        xt = torch.tensor(x, device="cuda:0", dtype=dtype)
        row = {}
        refs = {"iv": oracle.log_iv(v, x), "kv": oracle.log_kv(v, x)}     # once per set
        for fn in ("iv", "kv"):
            got = (B.log_iv if fn == "iv" else B.log_kv)(vt, xt).double().cpu().numpy()
            ref = refs[fn]
            e = oracle.rel_err(got, ref)
            i = int(np.argmax(e))
            row[fn] = {"max": float(e[i]), "p99": float(np.quantile(e, 0.99)), "at": [float(v[i]), float(x[i])]}
        fi, fk = B.log_ivkv(vt, xt)
        for nm, got, ref in (("ivkv_i", fi, refs["iv"]), ("ivkv_k", fk, refs["kv"])):
            e = oracle.rel_err(got.double().cpu().numpy(), ref)
            i = int(np.argmax(e))
            row[nm] = {"max": float(e[i]), "p99": float(np.quantile(e, 0.99)), "at": [float(v[i]), float(x[i])]}
        res[name] = row
        print(f"{name:10s} I max {row['iv']['max']:.2e} p99 {row['iv']['p99']:.1e} at {row['iv']['at']}   "
              f"K max {row['kv']['max']:.2e} p99 {row['kv']['p99']:.1e} at {row['kv']['at']}   "
              f"fused I {row['ivkv_i']['max']:.2e} K {row['ivkv_k']['max']:.2e} at {row['ivkv_k']['at']}", flush=True)
    return res


if __name__ == "__main__":
    # usage: python tools/accuracy_report.py [out.json] [points per set] [f32] [seed=S]
    dt = torch.float32 if "f32" in sys.argv[3:] else torch.float64
    sd = [int(a[5:]) for a in sys.argv[3:] if a.startswith("seed=")]
    r = main(int(sys.argv[2]), seed=sd[0] if sd else 0, dtype=dt) if len(sys.argv) > 2 else main()
    if len(sys.argv) > 1:
        json.dump(r, open(sys.argv[1], "w"), indent=1)
