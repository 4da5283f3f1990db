"""Seeded synthetic inputs shaped like the paper's workloads.

Shared by the tests, bench.py and the oracle legs; holds none of the method's
arithmetic (only random draws and grids).  Recipes:

* bench_grid      -- PAPER.md Fig. 1 caption (lines 33-35): v in {2^0..2^10},
                     20M x per v uniform in [1, 100]; laid out v-major
                     (all x for v=1, then v=2, ...), as the experiment sweeps v.
* small_case      -- BASELINE configs[0]: 10k pairs, integer v in 0..10,
                     x uniform in [1, 100].
* paper_region    -- §5.1-5.2 (lines 414-421): Small [0,150]^2, Large
                     [150,1e4]^2 (I) / [150,4000]^2 (K), uniform.
* stability_grid  -- BASELINE configs[3]: v in {0} U logspace(1e-3, 1e5),
                     x logspace(1e-3, 1e5), full outer product (Fig. 1b).
* vmf_features    -- §6.3 (lines 607-661): n unit-norm rows in R^d with a
                     prescribed mean resultant length (the CIFAR10/ResNet50
                     features of Table 7 have Rbar ~ 0.14-0.20).
"""
from __future__ import annotations

import math

import numpy as np
import torch

BENCH_ORDERS = tuple(float(2 ** j) for j in range(11))


def bench_grid(n_per_v: int = 20_000_000, seed: int = 0, device="cuda", dtype=torch.float64,
               orders=BENCH_ORDERS):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    nv = len(orders)
    v = torch.tensor(orders, dtype=dtype, device=device).repeat_interleave(n_per_v)
    x = torch.empty(nv * n_per_v, dtype=dtype, device=device)
    x.uniform_(1.0, 100.0, generator=g)
    return v, x


def bench_grid_slice(n_per_v: int, lo: int, hi: int, seed: int = 0, device="cuda", dtype=torch.float64,
                     orders=BENCH_ORDERS):
    """Elements [lo, hi) of ONE global v-major bench grid (the strong-scaling leg:
    every world size evaluates the same pairs).  The x of order j come from a
    generator seeded by (seed, j), so any contiguous slice is reproducible alone."""
    nv = len(orders)
    if not (0 <= lo <= hi <= nv * n_per_v):
        raise ValueError("slice out of range")
    vs, xs = [], []
    for j in range(lo // n_per_v, (hi + n_per_v - 1) // n_per_v if hi > lo else lo // n_per_v):
        a, b = max(lo, j * n_per_v), min(hi, (j + 1) * n_per_v)
        g = torch.Generator(device=device)
        g.manual_seed(seed * 1_000_003 + j + 1)
        x = torch.empty(n_per_v, dtype=dtype, device=device).uniform_(1.0, 100.0, generator=g)
        xs.append(x[a - j * n_per_v:b - j * n_per_v].clone())
        vs.append(torch.full((b - a,), orders[j], dtype=dtype, device=device))
        del x
    if not vs:
        return torch.empty(0, dtype=dtype, device=device), torch.empty(0, dtype=dtype, device=device)
    return torch.cat(vs), torch.cat(xs)


def bench_grid_numpy(n_per_v: int, seed: int = 0, orders=BENCH_ORDERS):
    rng = np.random.default_rng(seed)
    v = np.repeat(np.asarray(orders, dtype=np.float64), n_per_v)
    x = rng.uniform(1.0, 100.0, v.size)
    return v, x


def small_case(n: int = 10_000, seed: int = 0):
    rng = np.random.default_rng(seed)
    return rng.integers(0, 11, n).astype(np.float64), rng.uniform(1.0, 100.0, n)


def paper_region(n: int, region: str, fn: str = "iv", seed: int = 0):
    rng = np.random.default_rng(seed)
    if region == "small":
        lo, hi = 0.0, 150.0
    elif region == "large":
        lo, hi = 150.0, (1e4 if fn == "iv" else 4000.0)
    else:
        raise ValueError(region)
    return rng.uniform(lo, hi, n), rng.uniform(lo, hi, n)


def log_uniform(n: int, lo: float, hi: float, seed: int = 0):
    rng = np.random.default_rng(seed)
    return np.exp(rng.uniform(math.log(lo), math.log(hi), n))


def stability_axes(nv: int = 16384, nx: int = 16384):
    v = np.concatenate([[0.0], np.logspace(-3, 5, nv - 1)])
    x = np.logspace(-3, 5, nx)
    return v, x


def stability_grid(nv: int = 16384, nx: int = 16384, device="cuda", dtype=torch.float64, rows=None):
    """Outer product v x x (v-major).  `rows` = (r0, r1) selects a slice of v rows (sharding)."""
    va, xa = stability_axes(nv, nx)
    r0, r1 = (0, nv) if rows is None else rows
    vt = torch.tensor(va[r0:r1], dtype=dtype, device=device)
    xt = torch.tensor(xa, dtype=dtype, device=device)
    v = vt.repeat_interleave(nx)
    x = xt.repeat(r1 - r0)
    return v, x


def vmf_features(n: int, d: int, rbar: float = 0.15, seed: int = 0, device="cuda", dtype=torch.float32,
                 rows=None):
    """Rows x_i = normalize(c mu + z_i), z_i ~ N(0, I/d), c = rbar / sqrt(1 - rbar^2).

    The matrix is defined row-chunk by row-chunk: mu comes from `seed` alone and
    chunk k (a fixed number of rows for a given d) from its own generator
    seeded by (seed, k), so `rows=(lo, hi)` returns exactly rows lo..hi-1 of the
    full n x d matrix -- a rank's shard is a slice of the one matrix the N = 1
    run fits, whatever the world size.
    """
    lo, hi = (0, n) if rows is None else rows
    if not (0 <= lo <= hi <= n):
        raise ValueError("rows out of range")
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    mu = torch.randn(d, generator=g, device=device, dtype=torch.float64)
    mu /= mu.norm()
    c = rbar / math.sqrt(1.0 - rbar * rbar)
    X = torch.empty(hi - lo, d, device=device, dtype=dtype)
    chunk = max(1, (1 << 26) // (d * 8))
    for k in range(lo // chunk, (hi + chunk - 1) // chunk):
        a, b = k * chunk, min(n, (k + 1) * chunk)
        gk = torch.Generator(device=device)
        gk.manual_seed(seed * 1_000_003 + k + 1)
        z = torch.randn(b - a, d, generator=gk, device=device, dtype=torch.float64) / math.sqrt(d)
        z += c * mu
        z /= z.norm(dim=1, keepdim=True)
        s0, s1 = max(a, lo), min(b, hi)
        if s1 > s0:
            X[s0 - lo:s1 - lo] = z[s0 - a:s1 - a].to(dtype)
    return X, mu
