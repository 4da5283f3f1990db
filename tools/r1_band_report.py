"""Pure relative error of the f64 kernels where |log f| < 1 (R1), on a B200.

Parity tests measure |got - ref| / max(|ref|, 1).  This diagnostic reports, on the
log-uniform wide domain v, x in [1e-3, 1e5] plus a small-argument box v in [0, 1/2],
x in [1e-8, 2], the PURE relative error |got - ref| / |ref| of the points with
|ref| < 1, binned by |ref|, for log_iv / log_kv (separate) and the fused pass.  Near a
zero crossing of log f the pure relative error is ill-conditioned (the condition number
|x d(log f)/dx / log f| diverges), so large values in the smallest |ref| bins of K are
expected and are reported, not hidden.

  python tools/r1_band_report.py > profiles/<tag>/r1_band.json
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2409_08729_b200 as B  # noqa: E402
from paper_2409_08729_b200 import workloads  # noqa: E402


def main(n=400_000):
    dev = torch.device("cuda:0")
    v1 = workloads.log_uniform(n, 1e-3, 1e5, seed=1)
    x1 = workloads.log_uniform(n, 1e-3, 1e5, seed=2)
    rng = np.random.default_rng(3)
    v2 = rng.uniform(0.0, 0.5, n // 4)
    x2 = workloads.log_uniform(n // 4, 1e-8, 2.0, seed=4)
    v, x = np.concatenate([v1, v2]), np.concatenate([x1, x2])
    ri, rk = oracle.log_iv(v, x), oracle.log_kv(v, x)
    vt, xt = torch.tensor(v, device=dev), torch.tensor(x, device=dev)
    gi, gk = B.log_iv(vt, xt).cpu().numpy(), B.log_kv(vt, xt).cpu().numpy()
    fi, fk = (t.cpu().numpy() for t in B.log_ivkv(vt, xt))
    edges = [1.0, 1e-1, 1e-2, 1e-4, 1e-8, 0.0]
    out = {"points": int(v.size), "domain": "log-uniform v, x in [1e-3, 1e5] (400k) + v in [0, 1/2], "
                                           "x in [1e-8, 2] (100k)", "bins": {}}
    for name, got, ref in (("log_iv", gi, ri), ("log_kv", gk, rk), ("fused_I", fi, ri), ("fused_K", fk, rk)):
        d = {}
        for hi, lo in zip(edges, edges[1:]):
            m = (np.abs(ref) < hi) & (np.abs(ref) >= lo) & (ref != 0)
            if m.sum() == 0:
                continue
            e = np.abs(got[m] - ref[m]) / np.abs(ref[m])
            a = np.abs(got[m] - ref[m])
            d[f"[{lo:g},{hi:g})"] = {"n": int(m.sum()), "max_pure_rel": float(e.max()),
                                     "p99_pure_rel": float(np.quantile(e, 0.99)),
                                     "median_pure_rel": float(np.median(e)), "max_abs": float(a.max())}
        out["bins"][name] = d
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
