"""vMF fit timing on 50000 x d float32 features (diagnostic; bench.py reports the same in extra.vmf_fit).

Times (CUDA events, mean of reps): the column sum (partial + reduce, with the row-count
slot), the on-device scalar fit from the column sum, and the whole vmf_fit call.
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2409_08729_b200 as B  # noqa: E402
from paper_2409_08729_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:                 # diagnostic: time a variant build (tools/variant_bench.py)
    _lib.LIB = sys.argv[1]
from paper_2409_08729_b200 import workloads  # noqa: E402


def timed(f, reps=20):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3     # us


def main():
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6551.4
    out = {}
    for d in (2048, 8192, 32768):
        X, _ = workloads.vmf_features(50_000, d, rbar=0.15, seed=100, device="cuda:0")
        cs = torch.empty(d + 1, dtype=torch.float64, device="cuda:0")
        t_cs = timed(lambda: B.vmf_colsum(X, out=cs, with_count=True))
        t_fit = timed(lambda: B.vmf_fit_from_colsum(cs))
        t_all = timed(lambda: B.vmf_fit(X))
        mu, st = B.vmf_fit(X)
        gbs = X.numel() * 4 / (t_cs * 1e-6) / 1e9
        out[d] = {"colsum_us": t_cs, "fit_from_colsum_us": t_fit, "vmf_fit_us": t_all, "colsum_gbs": gbs,
                  "colsum_frac_hbm": gbs / peak, "iterations": float(st[7]), "kappa_mle": float(st[4])}
        del X
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
