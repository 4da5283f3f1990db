"""Dense f32 accuracy probe of the boxes with the thinnest margin (diagnostic, GPU box).

The 500k-point method-set runs (tools/accuracy_report.py) put the f32 maxima at the
edges of the eta band (the cancellation of rho + v log(x/(v+rho)) just outside it),
at the U13 / fallback edge and in the fallback band of log I alone.  This samples each
box with 1M points (inputs rounded to float, the oracle at those inputs) and prints
the max error of log I, log K and the fused pass per box.

  python tools/f32_probe.py [out.json] [points per box] [f64]   (f64: the f64 boxes)
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2409_08729_b200 as B  # noqa: E402

Z0 = 0.6627434193491816


def boxes(rng, n):
    lv = lambda a, b: np.exp(rng.uniform(np.log(a), np.log(b), n))   # noqa: E731
    v = lv(13.0, 2000.0)
    yield "eta_edge_lo", v, v * rng.uniform(Z0 - 0.16, Z0 - 0.10, n)
    v = lv(13.0, 2000.0)
    yield "eta_edge_hi", v, v * rng.uniform(Z0 + 0.10, Z0 + 0.16, n)
    yield "u13_fb_edge", rng.uniform(12.0, 16.0, n), rng.uniform(5.0, 12.0, n)
    yield "fb_b_high_v", rng.uniform(9.0, 12.69, n), rng.uniform(6.0, 19.69, n)
    yield "mu_corner", rng.uniform(10.0, 15.39, n), rng.uniform(30.0, 36.0, n)


def boxes64(rng, n):
    """f64: the U13 / fallback edge, the U term-count changes at rho = 61 / 107, the edges
    of the f64 eta band (0.03), the mu corner, U13 at small v just past x = 19.69."""
    lv = lambda a, b: np.exp(rng.uniform(np.log(a), np.log(b), n))   # noqa: E731
    yield "u13_fb_edge", rng.uniform(12.69, 14.0, n), rng.uniform(4.0, 12.0, n)
    for rho in (61.0, 107.0):
        r = rho * rng.uniform(1.0, 1.03, n)
        th = rng.uniform(0.0, np.pi / 2, n)
        yield f"rho{int(rho)}_edge", r * np.cos(th), r * np.sin(th)
    v = lv(13.0, 2000.0)
    yield "eta_edge", v, v * (Z0 + rng.choice([-1.0, 1.0], n) * rng.uniform(0.03, 0.05, n))
    yield "mu_corner", rng.uniform(10.0, 15.39, n), rng.uniform(30.0, 36.0, n)
    yield "u13_low_v", rng.uniform(0.7, 2.0, n), rng.uniform(19.69, 22.0, n)


def main(n=1_000_000, f64=False):
    rng = np.random.default_rng(11)
    res = {}
    dt = torch.float64 if f64 else torch.float32
    for name, v, x in (boxes64 if f64 else boxes)(rng, n):
        if not f64:
            v = v.astype(np.float32).astype(np.float64)
            x = x.astype(np.float32).astype(np.float64)
        vt = torch.tensor(v, device="cuda:0", dtype=dt)
        xt = torch.tensor(x, device="cuda:0", dtype=dt)
        ri, rk = oracle.log_iv(v, x), oracle.log_kv(v, x)
        fi, fk = B.log_ivkv(vt, xt)
        row = {}
        for what, got, ref in (("iv", B.log_iv(vt, xt), ri), ("kv", B.log_kv(vt, xt), rk),
                               ("ivkv_i", fi, ri), ("ivkv_k", fk, rk)):
            e = oracle.rel_err(got.double().cpu().numpy(), ref)
            i = int(np.argmax(e))
            row[what] = {"max": float(e[i]), "at": [float(v[i]), float(x[i])]}
        res[name] = row
        print(name, " ".join(f"{k} {r['max']:.2e}@({r['at'][0]:.4g},{r['at'][1]:.4g})" for k, r in row.items()),
              flush=True)
    return res


if __name__ == "__main__":
    r = main(int(sys.argv[2]), f64="f64" in sys.argv[3:]) if len(sys.argv) > 2 else main()
    if len(sys.argv) > 1:
        json.dump(r, open(sys.argv[1], "w"), indent=1)
