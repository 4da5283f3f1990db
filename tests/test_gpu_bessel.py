"""GPU parity: the CUDA path (through the C ABI) against the binary128 oracle.

Error measure: oracle.rel_err = |got - ref| / max(|ref|, 1)  (R1).
Bars: 1e-13 (f64) and 1e-5 (f32) from BASELINE.json north_star; 1e-8 for the
paper's own Simpson K fallback (its Table 2 reports 6.5e-9 in the Small region).
"""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2409_08729_b200 import workloads

pytestmark = pytest.mark.gpu

TOL64 = 1e-13
TOL32 = 1e-5


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2409_08729_b200 as B
    B.lib()
    return B


def _dev(a, dtype=torch.float64):
    return torch.tensor(np.asarray(a), dtype=dtype, device="cuda:0")


def _run(B, fn, v, x, dtype=torch.float64):
    f = {"iv": B.log_iv, "kv": B.log_kv, "kvp": B.log_kv_paper}[fn]
    out = f(_dev(v, dtype), _dev(x, dtype))
    torch.cuda.synchronize()
    return out.double().cpu().numpy()


def _ref(fn, v, x):
    return oracle.log_iv(v, x) if fn == "iv" else oracle.log_kv(v, x)


def _check(B, fn, v, x, tol=TOL64, dtype=torch.float64, what=""):
    got = _run(B, fn, v, x, dtype)
    if dtype == torch.float32:   # compare at the inputs the kernel actually saw
        v = np.asarray(v, np.float32).astype(np.float64)
        x = np.asarray(x, np.float32).astype(np.float64)
    ref = _ref("iv" if fn == "iv" else "kv", v, x)
    e = oracle.rel_err(got, ref)
    i = int(np.argmax(e)) if e.size else 0
    assert np.all(np.isfinite(got) | np.isinf(ref)), f"{what}: non-finite output"
    assert e.size == 0 or e[i] <= tol, f"{what} {fn}: max err {e[i]:.3e} at v={v[i]!r} x={x[i]!r} got={got[i]!r} ref={ref[i]!r}"
    return e


@pytest.mark.parametrize("fn", ["iv", "kv"])
def test_config0_small_case(B, fn):
    """BASELINE configs[0]: 10k pairs, integer v in 0..10, x ~ U[1,100]."""
    v, x = workloads.small_case(10_000, seed=0)
    _check(B, fn, v, x, what="configs[0]")


@pytest.mark.parametrize("fn", ["iv", "kv"])
@pytest.mark.parametrize("n", [0, 1, 7, 31, 1023, 1024, 1025, 4097, 65536 + 3])
def test_ragged_sizes(B, fn, n):
    """Tile (1024) and warp boundaries, empty input, mixed regions in one tile."""
    rng = np.random.default_rng(n)
    v = np.exp(rng.uniform(math.log(1e-3), math.log(2e3), n))
    x = np.exp(rng.uniform(math.log(1e-3), math.log(2e3), n))
    _check(B, fn, v, x, what=f"ragged n={n}")


@pytest.mark.parametrize("fn", ["iv", "kv"])
@pytest.mark.parametrize("region", ["small", "large"])
def test_paper_regions(B, fn, region):
    """PAPER.md §5.1 test regions (lines 414-416), uniform samples (§5.2)."""
    n = 20_000 if region == "small" else 4_000
    v, x = workloads.paper_region(n, region, fn, seed=11)
    _check(B, fn, v, x, what=f"{region} region")


@pytest.mark.parametrize("fn", ["iv", "kv"])
def test_region_boundaries(B, fn):
    """Points straddling every Table-1 threshold used on the GPU (lines 342-348)."""
    vs, xs = [], []
    eps = [-1e-9, 0.0, 1e-9]
    for xt in (30.0, 59.6925, 19.6931):
        for d in eps:
            for v in (0.0, 0.3, 0.7, 1.0, 5.0, 12.0, 15.3919, 20.0, 100.0):
                vs.append(v), xs.append(xt * (1 + d))
    for vt in (15.3919, 0.7, 12.6964):
        for d in eps:
            for x in (1e-3, 0.5, 5.0, 19.0, 25.0, 31.0, 70.0, 1e3):
                vs.append(vt * (1 + d)), xs.append(x)
    lx = np.linspace(math.log(60.0), math.log(1e5), 200)
    for l in lx:                                     # the curved mu-edge log v = 0.5113 log x + 0.7939
        vb = math.exp(0.5113 * l + 0.7939)
        for d in eps:
            vs.append(vb * (1 + d)), xs.append(math.exp(l))
    _check(B, fn, np.array(vs), np.array(xs), what="boundaries")


@pytest.mark.parametrize("fn", ["iv", "kv"])
def test_wide_domain(B, fn):
    """Log-uniform over the stability domain v in [1e-3, 1e5], x in [1e-3, 1e5]."""
    v = workloads.log_uniform(50_000, 1e-3, 1e5, seed=21)
    x = workloads.log_uniform(50_000, 1e-3, 1e5, seed=22)
    _check(B, fn, v, x, what="wide")


@pytest.mark.parametrize("fn", ["iv", "kv"])
def test_eta_root_band(B, fn):
    """x ~ 0.6627 v (eta(x/v) ~ 0, the Laplace limit) at large v: v*eta cancels."""
    v = workloads.log_uniform(20_000, 50.0, 1e5, seed=23)
    rng = np.random.default_rng(24)
    x = v * 0.66274341934918158 * (1 + rng.uniform(-0.1, 0.1, v.size))
    _check(B, fn, v, x, what="eta band")


@pytest.mark.parametrize("fn", ["iv", "kv"])
def test_f32(B, fn):
    v, x = workloads.small_case(10_000, seed=3)
    _check(B, fn, v, x, tol=TOL32, dtype=torch.float32, what="f32 configs[0]")
    v, x = workloads.paper_region(10_000, "small", fn, seed=4)
    _check(B, fn, v, x, tol=TOL32, dtype=torch.float32, what="f32 small")


def test_paper_k_integral(B):
    """The paper's Simpson fallback: parity at the paper's own accuracy (Table 2: 6.5e-9)."""
    v, x = workloads.paper_region(20_000, "small", "kv", seed=5)
    got = _run(B, "kvp", v, x)
    e = oracle.rel_err(got, oracle.log_kv(v, x))
    assert np.all(np.isfinite(got))
    assert e.max() <= 1e-8, e.max()


def test_special_values(B):
    v = np.array([0.0, 3.0, 0.0, 2.0, -1.0, 1.0, np.nan, 1.0, 20.0, 0.5])
    x = np.array([0.0, 0.0, 1e-300, -1.0, 2.0, np.nan, 1.0, np.inf, 0.0, 1e300])
    gi = _run(B, "iv", v, x)
    gk = _run(B, "kv", v, x)
    assert gi[0] == 0.0 and gi[1] == -np.inf and gi[8] == -np.inf
    assert np.isnan(gi[3]) and np.isnan(gi[4]) and np.isnan(gi[5]) and np.isnan(gi[6])
    assert gi[7] == np.inf
    assert np.isfinite(gi[2])
    assert gk[0] == np.inf and gk[1] == np.inf and gk[8] == np.inf
    assert np.isfinite(gk[4])                      # K_{-1} = K_1
    assert abs(gk[4] - oracle.log_kv(1.0, 2.0)) <= TOL64 * max(1, abs(gk[4]))
    assert np.isnan(gk[3]) and np.isnan(gk[5]) and np.isnan(gk[6])
    assert gk[7] == -np.inf
    assert np.isfinite(gi[9]) and np.isfinite(gk[9])


def test_negative_order_k(B):
    v = workloads.log_uniform(5000, 1e-3, 1e3, seed=8)
    x = workloads.log_uniform(5000, 1e-3, 1e3, seed=9)
    a = _run(B, "kv", -v, x)
    b = _run(B, "kv", v, x)
    assert np.array_equal(a, b)


def test_classify_matches_table1(B):
    """Dispatch is Algorithm 1 / Table 1 with the GPU branch set (bit-exact ids)."""
    rng = np.random.default_rng(12)
    v = np.concatenate([rng.uniform(0, 200, 50_000), [1.0, 200.0, 5.0, 1.0]])
    x = np.concatenate([rng.uniform(0, 200, 50_000), [1500.0, 10.0, 5.0, 1500.0]])
    got = B.classify(_dev(v), _dev(x)).cpu().numpy()

    # "a > C" is decided on IEEE high words: hi(a) > hi(C) (reading R3)
    def hw(a):
        return (np.asarray(a, np.float64).view(np.uint64) >> np.uint64(32)).astype(np.int64)

    def gt(a, c):
        return hw(a) > hw(c)
    with np.errstate(divide="ignore"):
        edge = (0.5113 * np.log(x) + 0.7939 > np.log(v)) | (hw(v) == 0)
    mu = (gt(x, 30.0) & ~gt(v, 15.3919)) | (edge & gt(x, 59.6925))
    u13 = (gt(x, 19.6931) & gt(v, 0.7)) | gt(v, 12.6964)
    want = np.where(mu, 0, np.where(u13, 1, 2))
    assert np.array_equal(got, want)
    assert list(got[-4:]) == [0, 1, 2, 0]     # SPEC.md dispatch examples in batch mode


def test_host_buffers_match_device(B):
    v, x = workloads.bench_grid_numpy(50_000, seed=4)
    a = B.log_iv_host(v, x)
    b = _run(B, "iv", v, x)
    assert np.array_equal(a, b)
    vt = torch.tensor(v).pin_memory()
    xt = torch.tensor(x).pin_memory()
    c = B.log_kv_host(vt, xt).numpy()
    d = _run(B, "kv", v, x)
    assert np.array_equal(c, d)


def test_deterministic(B):
    v, x = workloads.bench_grid_numpy(20_000, seed=5)
    assert np.array_equal(_run(B, "iv", v, x), _run(B, "iv", v, x))
    assert np.array_equal(_run(B, "kv", v, x), _run(B, "kv", v, x))


@pytest.mark.parametrize("fn", ["iv", "kv"])
def test_full_bench_grid_sampled(B, fn):
    """BASELINE configs[1]/[2] at full size (11 x 20M) in the bench launch
    configuration; all outputs finite, 20k sampled outputs against the oracle."""
    dev = torch.device("cuda:0")
    v, x = workloads.bench_grid(20_000_000, seed=0, device=dev)
    out = (B.log_iv if fn == "iv" else B.log_kv)(v, x)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(out).all())
    idx = torch.randint(0, v.numel(), (20_000,), generator=torch.Generator().manual_seed(1)).to(dev)
    vs, xs, gs = v[idx].cpu().numpy(), x[idx].cpu().numpy(), out[idx].cpu().numpy()
    e = oracle.rel_err(gs, _ref(fn, vs, xs))
    assert e.max() <= TOL64, e.max()
    del v, x, out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("fn", ["iv", "kv"])
def test_stability_sweep(B, fn):
    """BASELINE configs[3]: v in [0,1e5] x x in [1e-3,1e5] log-spaced, 16384^2 = 268M
    pairs: zero non-finite outputs; sampled outputs against the oracle."""
    dev = torch.device("cuda:0")
    total_bad = 0
    samples_v, samples_x, samples_g = [], [], []
    gen = torch.Generator().manual_seed(2)
    for r0 in range(0, 16384, 4096):
        v, x = workloads.stability_grid(16384, 16384, device=dev, rows=(r0, r0 + 4096))
        out = (B.log_iv if fn == "iv" else B.log_kv)(v, x)
        total_bad += int((~torch.isfinite(out)).sum().item())
        idx = torch.randint(0, v.numel(), (1500,), generator=gen).to(dev)
        samples_v.append(v[idx].cpu().numpy()), samples_x.append(x[idx].cpu().numpy())
        samples_g.append(out[idx].cpu().numpy())
        del v, x, out
    torch.cuda.empty_cache()
    # only x = 1e-3.. > 0 and v >= 0 in this grid: every output must be finite
    assert total_bad == 0
    vs, xs, gs = map(np.concatenate, (samples_v, samples_x, samples_g))
    e = oracle.rel_err(gs, _ref(fn, vs, xs))
    assert e.max() <= TOL64, e.max()


# ------------------------------------------------------------------ fused I + K
def _run_ivkv(B, v, x, dtype=torch.float64):
    oi, ok = B.log_ivkv(_dev(v, dtype), _dev(x, dtype))
    torch.cuda.synchronize()
    return oi.double().cpu().numpy(), ok.double().cpu().numpy()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("case", ["config0", "ragged", "wide", "eta", "fallback_band", "temme_band", "special"])
def test_fused_ivkv_against_oracle(B, case):
    """b200_log_ivkv_f64: both functions in one pass, each within the f64 bar."""
    if case == "config0":
        v, x = workloads.small_case(10_000, seed=30)
    elif case == "ragged":
        rng = np.random.default_rng(31)
        v = np.exp(rng.uniform(math.log(1e-3), math.log(2e3), 4097))
        x = np.exp(rng.uniform(math.log(1e-3), math.log(2e3), 4097))
    elif case == "wide":
        v = workloads.log_uniform(30_000, 1e-3, 1e5, seed=32)
        x = workloads.log_uniform(30_000, 1e-3, 1e5, seed=33)
    elif case == "fallback_band":
        # 2 < x <= 30, v <= 12.7: the fused pass takes log I from the K values
        # (Wronskian + Miller ratio); edges of the band included
        rng = np.random.default_rng(37)
        v = rng.uniform(0.0, 12.69, 20_000)
        x = rng.uniform(2.0, 30.0, 20_000)
        v[:8] = [0.0, 0.5, 0.4999, 12.69, 12.5, 1.0, 0.7, 0.0]
        x[:8] = [2.000001, 30.0, 2.5, 2.000001, 19.69, 19.7, 29.99, 29.99]
    elif case == "temme_band":
        # x <= 2, v <= 12.7: for 1e-6 <= x the fused pass takes log I from
        # Temme's K values (Wronskian + Miller ratio); below 1e-6 the series
        rng = np.random.default_rng(38)
        v = rng.uniform(0.0, 12.69, 20_000)
        x = workloads.log_uniform(20_000, 1e-8, 2.0, seed=39)
        v[:6] = [0.0, 0.5, 12.69, 12.69, 0.0, 7.3]
        x[:6] = [1e-6, 2.0, 1e-6, 2.0, 0.999999e-6, 1.0000001e-6]
    elif case == "eta":
        v = workloads.log_uniform(10_000, 50.0, 1e5, seed=34)
        x = v * 0.66274341934918158 * (1 + np.random.default_rng(35).uniform(-0.1, 0.1, v.size))
    else:
        v = np.array([0.0, 3.0, 0.0, 2.0, -1.0, 1.0, 1.0, 20.0, 0.5, 1e150, 5.0])
        x = np.array([0.0, 0.0, 1e-300, -1.0, 2.0, np.nan, np.inf, 0.0, 1e300, 3.0, 1e-200])
    gi, gk = _run_ivkv(B, v, x)
    si = _run(B, "iv", v, x)
    sk = _run(B, "kv", v, x)
    # same special values / NaN pattern as the separate calls
    assert np.array_equal(np.isnan(gi), np.isnan(si)) and np.array_equal(np.isnan(gk), np.isnan(sk))
    assert np.array_equal(np.isinf(gi), np.isinf(si)) and np.array_equal(np.isinf(gk), np.isinf(sk))
    if case == "special":      # extreme arguments: agree with the separate calls (no oracle run)
        ok = np.isfinite(si) & np.isfinite(sk)
        assert oracle.rel_err(gi[ok], si[ok]).max() <= TOL64 and oracle.rel_err(gk[ok], sk[ok]).max() <= TOL64
        return
    ok = np.isfinite(si) & np.isfinite(sk)
    ri = oracle.log_iv(np.abs(v[ok]), x[ok])
    rk = oracle.log_kv(v[ok], x[ok])
    assert oracle.rel_err(gi[ok], ri).max() <= TOL64
    assert oracle.rel_err(gk[ok], rk).max() <= TOL64


# pairs per tile of the f64 fused pass: KTile<double, FN_IK>::tile = TPB * B200_SB_ITEMS
# (bessel_kernels.cu; tests/test_tile_logic.py checks the source against this value)
FUSED_TILE = 256 * 11

# one (v, x) box per evaluation bin of the fused pass (R12/R13, Table 1 predicates)
_BIN_BOXES = {
    "mu": ((0.0, 10.0), (40.0, 90.0)),
    "u6": ((300.0, 800.0), (1.0, 100.0)),
    "u8": ((120.0, 250.0), (1.0, 100.0)),
    "u10": ((65.0, 100.0), (1.0, 60.0)),
    "u13": ((14.0, 50.0), (1.0, 19.0)),
    "temme": ((0.5, 12.0), (0.1, 2.0)),
    "trapezoid": ((0.5, 12.0), (2.5, 19.0)),
    "slow": ((0.0, 5.0), (1e-150, 1e-145)),      # x below the f64 operating range (R13)
}


@pytest.mark.timeout(600)
def test_fused_every_bin_in_every_tile(B):
    """Mixed tiles of the fused f64 pass (costliest-first order, bins padded to 32-slot
    chunks, snake dealing): every tile holds all eight bins, with per-bin
    counts of 0, 1, 31, 32, 33 and more (no padding, 31 padding slots, a bin that fills
    whole chunks), shuffled, plus a ragged last tile; both results against the oracle."""
    rng = np.random.default_rng(41)
    counts = [[32, 1, 31, 33, 64, 5, 17, 3], [0, 200, 0, 0, 1, 0, 100, 0], [1, 1, 1, 1, 1, 1, 1, 1],
              [192, 0, 64, 0, 96, 31, 33, 32], [7, 40, 9, 300, 2, 11, 5, 1]]
    names = list(_BIN_BOXES)
    vs, xs = [], []
    for row in counts + [[9, 9, 9, 9, 9, 9, 9, 9]]:          # the last tile is ragged (72 pairs)
        tv, tx = [], []
        for nm, c in zip(names, row):
            (v0, v1), (x0, x1) = _BIN_BOXES[nm]
            tv.append(rng.uniform(v0, v1, c))
            tx.append(np.exp(rng.uniform(math.log(x0), math.log(x1), c)) if nm == "slow" else rng.uniform(x0, x1, c))
        tv, tx = np.concatenate(tv), np.concatenate(tx)
        if len(vs) < len(counts):                  # fill the full tiles with mu pairs
            k = FUSED_TILE - tv.size
            tv = np.concatenate([tv, rng.uniform(0.0, 10.0, k)])
            tx = np.concatenate([tx, rng.uniform(40.0, 90.0, k)])
        perm = rng.permutation(tv.size)
        vs.append(tv[perm])
        xs.append(tx[perm])
    v, x = np.concatenate(vs), np.concatenate(xs)
    assert v.size == 5 * FUSED_TILE + 72
    gi, gk = _run_ivkv(B, v, x)
    assert np.all(np.isfinite(gi)) and np.all(np.isfinite(gk))
    ri, rk = oracle.log_iv(v, x), oracle.log_kv(v, x)
    ei, ek = oracle.rel_err(gi, ri), oracle.rel_err(gk, rk)
    i, k = int(np.argmax(ei)), int(np.argmax(ek))
    assert ei[i] <= TOL64, f"log I err {ei[i]:.3e} at v={v[i]!r} x={x[i]!r}"
    assert ek[k] <= TOL64, f"log K err {ek[k]:.3e} at v={v[k]!r} x={x[k]!r}"


def test_fused_ivkv_f32_and_host(B):
    v, x = workloads.small_case(10_000, seed=36)
    gi, gk = _run_ivkv(B, v, x, torch.float32)
    v32 = np.asarray(v, np.float32).astype(np.float64)
    x32 = np.asarray(x, np.float32).astype(np.float64)
    assert oracle.rel_err(gi, oracle.log_iv(v32, x32)).max() <= TOL32
    assert oracle.rel_err(gk, oracle.log_kv(v32, x32)).max() <= TOL32
    v, x = workloads.bench_grid_numpy(30_000, seed=37)
    hi, hk = B.log_ivkv_host(v, x)
    di, dk = _run_ivkv(B, v, x)
    assert np.array_equal(hi, di) and np.array_equal(hk, dk)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_unaligned_pointers_use_the_cp_async_path(B, dtype):
    """Views starting one element into an allocation are not 16-byte aligned: the
    kernel falls back from bulk (TMA) copies to per-thread cp.async; same results."""
    v, x = workloads.bench_grid_numpy(3000, seed=40)
    vt = torch.tensor(np.concatenate([[1.0], v]), dtype=dtype, device="cuda:0")
    xt = torch.tensor(np.concatenate([[1.0], x]), dtype=dtype, device="cuda:0")
    va, xa = vt[1:], xt[1:]
    assert va.data_ptr() % 16 != 0
    outs = torch.empty(v.size + 1, dtype=dtype, device="cuda:0")[1:]
    for fn in (B.log_iv, B.log_kv):
        got = fn(va, xa, out=outs).clone()
        ref = fn(va.clone(), xa.clone())
        assert torch.equal(got, ref)
    gi, gk = B.log_ivkv(va, xa)
    ri, rk = B.log_ivkv(va.clone(), xa.clone())
    assert torch.equal(gi, ri) and torch.equal(gk, rk)
    if dtype == torch.float64:
        e = oracle.rel_err(gi.cpu().numpy(), oracle.log_iv(v, x))
        assert e.max() <= TOL64


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_unaligned_pointers_over_several_waves(B, dtype):
    """More tiles than resident CTAs (148 SMs x 4-6 CTAs x 2816 pairs), so every CTA
    reloads its single stage: the cp.async path (unaligned views) must give the same
    bits as the bulk-copy path, for all three entry points and a ragged last tile."""
    n = 2 * 148 * 6 * FUSED_TILE + 1235
    v, x = workloads.bench_grid(n // 11 + 1, seed=45, device="cuda:0", dtype=dtype)
    v, x = v[:n].contiguous(), x[:n].contiguous()
    vt = torch.empty(n + 1, dtype=dtype, device="cuda:0")
    xt = torch.empty(n + 1, dtype=dtype, device="cuda:0")
    vt[1:].copy_(v)
    xt[1:].copy_(x)
    va, xa = vt[1:], xt[1:]
    assert va.data_ptr() % 16 != 0
    for fn in (B.log_iv, B.log_kv):
        assert torch.equal(fn(va, xa), fn(v, x))
    gi, gk = B.log_ivkv(va, xa)
    ri, rk = B.log_ivkv(v, x)
    assert torch.equal(gi, ri) and torch.equal(gk, rk)


def test_tile_tails_against_separate_sizes(B):
    """Every tail length of the last tile (bulk part + < 2 leftover elements)."""
    v, x = workloads.bench_grid_numpy(400, seed=41)
    full_i = _run(B, "iv", v, x)
    for n in (1, 2, 3, 1023, 1025, 2047, 2049, 3001):
        got = _run(B, "iv", v[:n], x[:n])
        assert np.array_equal(got, full_i[:n]), n


@pytest.mark.parametrize("fn", ["iv", "kv"])
def test_tiny_arguments_stay_finite(B, fn):
    """x down to the smallest subnormal with orders up to the fallback edge: log K ~ v log(2/x)
    is finite (scaled forward recurrence below x = 1e-6), every point against the oracle."""
    xs = np.array([5e-324, 1e-310, 1e-300, 1e-200, 1e-141, 1e-139, 1e-100, 1e-30, 1e-8, 9.9e-7, 1.01e-6])
    vs = np.array([0.0, 0.3, 1.0, 5.0, 5.5, 12.0, 12.6])
    v, x = np.meshgrid(vs, xs)
    v, x = v.ravel(), x.ravel()
    got = _run(B, fn, v, x)
    assert np.all(np.isfinite(got) | ((fn == "iv") & (v > 0) & np.isinf(got) & (got < 0)))
    ok = np.ones(v.size, bool)                     # the oracle evaluates all of these (binary128)
    ref = _ref(fn, v[ok], x[ok])
    assert oracle.rel_err(got[ok], ref).max() <= TOL64


def test_full_bench_grid_fused_sampled(B):
    """The bench step itself: b200_log_ivkv_f64 over the full configs[1]/[2] grid
    (11 x 20M pairs) in the bench launch configuration; all outputs finite, 20k
    sampled pairs of both results against the oracle."""
    dev = torch.device("cuda:0")
    v, x = workloads.bench_grid(20_000_000, seed=0, device=dev)
    oi, ok = B.log_ivkv(v, x)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(oi).all()) and bool(torch.isfinite(ok).all())
    idx = torch.randint(0, v.numel(), (20_000,), generator=torch.Generator().manual_seed(3)).to(dev)
    vs, xs = v[idx].cpu().numpy(), x[idx].cpu().numpy()
    assert oracle.rel_err(oi[idx].cpu().numpy(), oracle.log_iv(vs, xs)).max() <= TOL64
    assert oracle.rel_err(ok[idx].cpu().numpy(), oracle.log_kv(vs, xs)).max() <= TOL64
    del v, x, oi, ok
    torch.cuda.empty_cache()


def test_c_abi_from_plain_c(B, tmp_path):
    """The shared library used from C (tools/capi_example.c): device and host-buffer
    entry points against the half-integer closed forms, argument errors reported."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2409_08729_b200", "lib")
    exe = str(tmp_path / "capi_example")
    subprocess.check_call(["nvcc", "-Wno-deprecated-gpu-targets", "-o", exe,
                           os.path.join(root, "tools", "capi_example.c"),
                           "-I" + os.path.join(root, "include"), "-L" + libdir, "-lbessel_b200",
                           "-Xlinker", "-rpath=" + libdir])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "max rel err" in r.stdout


def test_fused_deterministic_and_on_side_stream(B):
    """Same inputs, same bits (fixed per-element evaluation order); the kernels run on
    the caller's current stream (a side stream here) and honour its ordering."""
    v, x = workloads.bench_grid_numpy(20_000, seed=42)
    vt, xt = _dev(v), _dev(x)
    a = B.log_ivkv(vt, xt)
    b = B.log_ivkv(vt, xt)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        vs, xs = vt.clone(), xt.clone()        # produced on the side stream
        c = B.log_ivkv(vs, xs)
        ci = B.log_iv(vs, xs)
    s.synchronize()
    assert torch.equal(c[0], a[0]) and torch.equal(c[1], a[1])
    assert oracle.rel_err(ci.cpu().numpy(), oracle.log_iv(v, x)).max() <= TOL64


@pytest.mark.timeout(600)
def test_more_than_2_pow_31_pairs(B):
    """n = 2^31 + 4097 pairs in one fused f64 call (69 GB of operands): element
    and tile offsets past the 32-bit range.  Sampled outputs -- both sides of
    2^31, the ragged last tile and random positions -- against the oracle, and
    the same samples re-evaluated in a small call (results depend only on
    (v_i, x_i), include/bessel_b200.h)."""
    dev = torch.device("cuda:0")
    n = 2 ** 31 + 4097
    free, _ = torch.cuda.mem_get_info(dev)
    if free < 4 * 8 * n + (8 << 30):
        pytest.skip(f"needs {4 * 8 * n / 2**30:.0f} GiB free device memory")
    g = torch.Generator(device=dev).manual_seed(11)
    v = torch.empty(n, dtype=torch.float64, device=dev).uniform_(0.0, 60.0, generator=g)
    x = torch.empty(n, dtype=torch.float64, device=dev).uniform_(1e-2, 120.0, generator=g)
    oi, ok = B.log_ivkv(v, x)
    torch.cuda.synchronize()
    edge = torch.arange(-2048, 2048, device=dev) + 2 ** 31
    tail = torch.arange(n - 2048, n, device=dev)
    rnd = torch.randint(0, n, (4000,), generator=torch.Generator().manual_seed(5)).to(dev)
    idx = torch.cat([edge, tail, rnd])
    vs, xs = v[idx].clone(), x[idx].clone()
    gi, gk = oi[idx].cpu().numpy(), ok[idx].cpu().numpy()
    del v, x, oi, ok
    torch.cuda.empty_cache()
    si, sk = B.log_ivkv(vs, xs)
    assert np.array_equal(si.cpu().numpy(), gi) and np.array_equal(sk.cpu().numpy(), gk)
    vn, xn = vs.cpu().numpy(), xs.cpu().numpy()
    assert oracle.rel_err(gi, oracle.log_iv(vn, xn)).max() <= TOL64
    assert oracle.rel_err(gk, oracle.log_kv(vn, xn)).max() <= TOL64


# ------------------------------------------------------------------ f32 coverage (configs[2] fp32 variant)
def _bin_counts(B, v, x):
    from paper_2409_08729_b200 import gen_tables
    th = gen_tables.u_term_thresholds()
    reg = B.classify(_dev(v), _dev(x)).cpu().numpy()
    m = np.maximum(v, x)
    names = {
        "mu": reg == 0,
        "U6": (reg == 1) & (m >= th[6]),
        "U8": (reg == 1) & (m < th[6]) & (m >= th[8]),
        "U10": (reg == 1) & (m < th[8]) & (m >= th[10]),
        "U13": (reg == 1) & (m < th[10]),
        "fallback x<=2": (reg == 2) & (x <= 2.0),
        "fallback x>2": (reg == 2) & (x > 2.0),
    }
    return {k: int(a.sum()) for k, a in names.items()}


def _f32_inputs(case):
    if case == "bench_grid":
        v, x = workloads.bench_grid_numpy(6000, seed=50)
    elif case == "large":
        v, x = workloads.paper_region(30_000, "large", "iv", seed=51)
    else:
        v = workloads.log_uniform(60_000, 1e-3, 1e5, seed=52)
        x = workloads.log_uniform(60_000, 1e-3, 1e5, seed=53)
    return np.asarray(v, np.float32).astype(np.float64), np.asarray(x, np.float32).astype(np.float64)


@pytest.mark.parametrize("case", ["bench_grid", "large", "wide"])
def test_f32_against_oracle(B, case):
    """fp32 variant of both kernels and of the fused pass at 1e-5 (north_star) on the
    fp32 bench grid (sampled), the paper's Large region and the log-uniform wide domain;
    every f32 evaluation bin (mu, U6, U8, U10, U13, both fallback classes) is hit."""
    v, x = _f32_inputs(case)
    cnt = _bin_counts(B, v, x)
    need = {"bench_grid": ["mu", "U6", "U8", "U10", "U13", "fallback x<=2", "fallback x>2"],
            "large": ["mu", "U6"],
            "wide": ["mu", "U6", "U8", "U10", "U13", "fallback x<=2", "fallback x>2"]}[case]
    for k in need:
        assert cnt[k] >= 50, (case, cnt)
    ri, rk = oracle.log_iv(v, x), oracle.log_kv(v, x)
    gi = _run(B, "iv", v, x, torch.float32)
    gk = _run(B, "kv", v, x, torch.float32)
    fi, fk = _run_ivkv(B, v, x, torch.float32)
    for name, got, ref in (("log_iv_f32", gi, ri), ("log_kv_f32", gk, rk), ("fused I f32", fi, ri),
                           ("fused K f32", fk, rk)):
        assert np.all(np.isfinite(got)), name
        e = oracle.rel_err(got, ref)
        i = int(np.argmax(e))
        assert e[i] <= TOL32, f"{case} {name}: {e[i]:.3e} at v={v[i]!r} x={x[i]!r}"


def test_f32_full_bench_grid_sampled(B):
    """configs[2] fp32 variant at full size (11 x 20M pairs, float32, the bench's fp32 leg):
    all outputs finite, 20k sampled pairs of the separate and fused passes against the oracle."""
    dev = torch.device("cuda:0")
    v, x = workloads.bench_grid(20_000_000, seed=0, device=dev, dtype=torch.float32)
    oi, ok = B.log_ivkv(v, x)
    si = B.log_iv(v, x)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(oi).all()) and bool(torch.isfinite(ok).all()) and bool(torch.isfinite(si).all())
    idx = torch.randint(0, v.numel(), (20_000,), generator=torch.Generator().manual_seed(9)).to(dev)
    vs, xs = v[idx].double().cpu().numpy(), x[idx].double().cpu().numpy()
    ri, rk = oracle.log_iv(vs, xs), oracle.log_kv(vs, xs)
    assert oracle.rel_err(oi[idx].double().cpu().numpy(), ri).max() <= TOL32
    assert oracle.rel_err(ok[idx].double().cpu().numpy(), rk).max() <= TOL32
    assert oracle.rel_err(si[idx].double().cpu().numpy(), ri).max() <= TOL32
    del si
    sk = B.log_kv(v, x)
    assert oracle.rel_err(sk[idx].double().cpu().numpy(), rk).max() <= TOL32
    del v, x, oi, ok, sk
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ the slow bin (outside the operating range)
TINY64 = [1e-141, 1e-150, 1e-200, 1e-300, 1e-310, 5e-324]
TINY32 = [1e-19, 1e-25, 1e-30, 1e-39, 1.4e-45]
ORDERS_SMALLX = [0.0, 0.3, 0.5, 1.0, 5.0, 5.5, 12.0, 12.6, 20.0, 100.0]


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_slow_bin_tiny_arguments_against_oracle(B, dtype):
    """x below the fast paths' range (1e-140 f64, 1e-18 f32), subnormals included: the slow
    bin (library log, scaled forward recurrence for K, log(x/2) without forming x/2) against
    the binary128 oracle, separate and fused passes."""
    xs = TINY64 if dtype == torch.float64 else TINY32
    v, x = np.meshgrid(ORDERS_SMALLX, xs)
    v, x = v.ravel(), x.ravel()
    if dtype == torch.float32:
        v = v.astype(np.float32).astype(np.float64)
        x = x.astype(np.float32).astype(np.float64)
    tol = TOL64 if dtype == torch.float64 else TOL32
    ri, rk = oracle.log_iv(v, x), oracle.log_kv(v, x)
    gi, gk = _run(B, "iv", v, x, dtype), _run(B, "kv", v, x, dtype)
    fi, fk = _run_ivkv(B, v, x, dtype)
    fin32 = np.abs(ri) < 3e38 if dtype == torch.float32 else np.ones(v.size, bool)
    for name, got, ref in (("iv", gi, ri), ("kv", gk, rk), ("fused I", fi, ri), ("fused K", fk, rk)):
        ok = fin32 & np.isfinite(ref)
        assert np.all(np.isfinite(got[ok])), (name, v[ok][~np.isfinite(got[ok])], x[ok][~np.isfinite(got[ok])])
        e = oracle.rel_err(got[ok], ref[ok])
        i = int(np.argmax(e))
        assert e[i] <= tol, f"{name}: {e[i]:.3e} at v={v[ok][i]!r} x={x[ok][i]!r} got={got[ok][i]!r} ref={ref[ok][i]!r}"


def _mp_log_iv_kv(v, x):
    import mpmath
    mpmath.mp.dps = 40
    return float(mpmath.log(mpmath.besseli(v, x))), float(mpmath.log(mpmath.besselk(v, x)))


def _debye_leading(v, x):
    """Leading term of the uniform expansion (DLMF 10.41.3/10.41.4) in 40-digit arithmetic:
    for v >= 1e19 the omitted u_1(t)/v term is < 1e-20 relative -- exact at f64 resolution."""
    import mpmath
    mpmath.mp.dps = 60
    V, X = mpmath.mpf(v), mpmath.mpf(x)
    z = X / V
    s = mpmath.sqrt(1 + z * z)
    eta = s + mpmath.log(z / (1 + s))
    base = -mpmath.log(s) / 2
    li = -mpmath.log(2 * mpmath.pi * V) / 2 + V * eta + base
    lk = mpmath.log(mpmath.pi / (2 * V)) / 2 - V * eta + base
    return float(li), float(lk)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_slow_bin_huge_arguments(B, dtype):
    """x or v above the fast range (1e140 f64, 1e18 f32).  The binary128 oracle cannot
    evaluate these (a series of ~x terms / an integrand peak narrower than its bracket), so
    the references are independent ones: mpmath besseli/besselk at 40 digits for huge x,
    the leading uniform-expansion term (exact to < 1e-20 relative there) for huge v.
    Includes the f32 case v = 2e19, x = 1 (v^2 + x^2 would overflow a float)."""
    if dtype == torch.float64:
        px = [(0.0, 1e141), (1.0, 1e150), (50.0, 1e200), (1e3, 1e300)]
        pv = [(1e141, 1.0), (1e200, 1e100), (1e300, 1e141), (2e150, 3e150)]
        tol = TOL64
    else:
        px = [(0.0, 1e19), (1.0, 1e30), (50.0, 3e37)]
        pv = [(2e19, 1.0), (1e30, 1e19), (1e25, 3e25), (1e20, 1e-3)]
        tol = TOL32
    v = np.array([p[0] for p in px + pv])
    x = np.array([p[1] for p in px + pv])
    if dtype == torch.float32:
        v = v.astype(np.float32).astype(np.float64)
        x = x.astype(np.float32).astype(np.float64)
    refs = [_mp_log_iv_kv(a, b) for a, b in zip(v[:len(px)], x[:len(px)])] + \
           [_debye_leading(a, b) for a, b in zip(v[len(px):], x[len(px):])]
    ri = np.array([r[0] for r in refs])
    rk = np.array([r[1] for r in refs])
    gi, gk = _run(B, "iv", v, x, dtype), _run(B, "kv", v, x, dtype)
    fi, fk = _run_ivkv(B, v, x, dtype)
    for name, got, ref in (("iv", gi, ri), ("kv", gk, rk), ("fused I", fi, ri), ("fused K", fk, rk)):
        assert np.all(np.isfinite(got)), (name, got)
        e = oracle.rel_err(got, ref)
        i = int(np.argmax(e))
        assert e[i] <= tol, f"{name}: {e[i]:.3e} at v={v[i]!r} x={x[i]!r} got={got[i]!r} ref={ref[i]!r}"


def test_pure_relative_accuracy_where_log_iv_is_small(B):
    """DESIGN.md R1: parity uses |got - ref| / max(|ref|, 1).  Where log I_v(x) itself is
    small but not at a zero crossing -- v < 1/2 and x <= 1/2 (log I_0(x) ~ x^2/4 down to
    1e-17) -- the series carries sum - 1 and log1p's, so the PURE relative error
    |got - ref| / |ref| holds 1e-13 too, in the separate and the fused pass."""
    rng = np.random.default_rng(61)
    v = np.concatenate([np.zeros(2000), rng.uniform(0.0, 0.4999, 8000)])
    x = workloads.log_uniform(10_000, 1e-8, 0.5, seed=62)
    ref = oracle.log_iv(v, x)
    gi = _run(B, "iv", v, x)
    fi, _ = _run_ivkv(B, v, x)
    nz = ref != 0.0
    for name, got in (("log_iv", gi), ("fused I", fi)):
        e = np.abs(got[nz] - ref[nz]) / np.abs(ref[nz])
        i = int(np.argmax(e))
        assert e[i] <= TOL64, f"{name}: pure rel err {e[i]:.3e} at v={v[nz][i]!r} x={x[nz][i]!r}"
    assert np.all(np.abs(gi[~nz]) <= 1e-300)


def test_mu_corner_cancellation(B):
    """The corner of the mu region (x just above 30, v up to 15.39: Table 1) is where the
    series for I alternates and cancels most (terms up to ~9 summing to ~0.02).  f32 must
    stay inside its bar there for both entry points -- the fused pass once summed S_I as
    E - O in float and reached 1.06e-5 (profiles/r165) -- and f64 inside its own."""
    rng = np.random.default_rng(47)
    n = 100_000
    v = rng.uniform(12.0, 15.39, n)
    x = rng.uniform(30.0, 32.0, n)
    for dtype, tol in ((torch.float32, TOL32), (torch.float64, TOL64)):
        if dtype == torch.float32:
            vv = v.astype(np.float32).astype(np.float64)
            xx = x.astype(np.float32).astype(np.float64)
        else:
            vv, xx = v, x
        ri, rk = oracle.log_iv(vv, xx), oracle.log_kv(vv, xx)
        gi, gk = _run_ivkv(B, vv, xx, dtype)
        si = _run(B, "iv", vv, xx, dtype)
        for got, ref, what in ((gi, ri, "fused I"), (gk, rk, "fused K"), (si, ri, "log_iv")):
            e = oracle.rel_err(got, ref)
            i = int(np.argmax(e))
            assert e[i] <= tol, f"{dtype} {what}: {e[i]:.3e} at v={vv[i]!r} x={xx[i]!r}"


def test_fused_f32_temme_band(B):
    """f32 fused pass on 0.1 <= x <= 2, 1/2 <= v <= 12.7, where log I comes from Temme's K values
    by the Wronskian and Miller's ratio (float range: the ratio is formed before the product
    with K_{v+1}/K_mu, which alone reaches ~1e27 at x = 0.1); edges of the band included."""
    rng = np.random.default_rng(63)
    v = rng.uniform(0.5, 12.69, 20_000)
    x = workloads.log_uniform(20_000, 0.05, 2.0, seed=64)
    v[:8] = [12.69, 12.69, 0.5, 0.5, 7.3, 12.69, 0.5, 3.0]
    x[:8] = [0.1, 0.0999, 0.1, 2.0, 0.1000001, 2.0, 0.0999, 1.0]
    v = v.astype(np.float32).astype(np.float64)
    x = x.astype(np.float32).astype(np.float64)
    gi, gk = _run_ivkv(B, v, x, torch.float32)
    assert np.all(np.isfinite(gi)) and np.all(np.isfinite(gk))
    ri, rk = oracle.log_iv(v, x), oracle.log_kv(v, x)
    for name, got, ref in (("I", gi, ri), ("K", gk, rk)):
        e = oracle.rel_err(got, ref)
        i = int(np.argmax(e))
        assert e[i] <= TOL32, f"fused f32 {name}: {e[i]:.3e} at v={v[i]!r} x={x[i]!r}"
