"""GPU parity of the vMF fit (§6.3) against oracle/vmf.py."""
import math

import numpy as np
import pytest
import torch

import oracle
from oracle import vmf as ovmf
from paper_2409_08729_b200 import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2409_08729_b200 as B
    B.lib()
    return B


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("n,d", [(1, 2), (3, 5), (1000, 64), (4097, 1030), (777, 2048)])
def test_colsum_exact(B, dtype, n, d):
    X, _ = workloads.vmf_features(n, d, rbar=0.4, seed=n + d, device="cuda:0", dtype=dtype)
    got = B.vmf_colsum(X).cpu().numpy()
    Xh = X.double().cpu().numpy()
    ref = np.array([math.fsum(Xh[:, j]) for j in range(d)])
    assert np.max(np.abs(got - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref))) + 1e-15 * n


def test_colsum_strided_and_accumulate(B):
    X, _ = workloads.vmf_features(513, 300, seed=1, device="cuda:0", dtype=torch.float32)
    big = torch.zeros(513, 301, device="cuda:0", dtype=torch.float32)
    big[:, :300] = X
    view = big[:, :300]                      # ld = 301, not 16-byte aligned rows
    a = B.vmf_colsum(view)
    b = B.vmf_colsum(X)
    assert torch.allclose(a, b, rtol=0, atol=1e-12)
    c = B.vmf_colsum(X, out=b.clone(), accumulate=True)
    assert torch.allclose(c, 2 * b, rtol=1e-15, atol=0)


@pytest.mark.parametrize("d,rbar", [(64, 0.7), (256, 0.3), (2048, 0.15), (8192, 0.19), (2048, 0.95)])
def test_fit_against_oracle(B, d, rbar):
    X, _ = workloads.vmf_features(3000, d, rbar=rbar, seed=d, device="cuda:0", dtype=torch.float64)
    mu, stats = B.vmf_fit(X)
    s = stats.cpu().numpy()
    ref = ovmf.fit(X.cpu().numpy())
    assert abs(s[0] - ref["rbar"]) <= 1e-13
    assert np.max(np.abs(mu.cpu().numpy() - ref["mu"])) <= 1e-12
    assert abs(s[1] - ref["kappa0"]) <= 1e-12 * ref["kappa0"]
    # kappa1 = F(kappa0), kappa2 = F(kappa1), kappa_mle = A_p^{-1}(Rbar).  All
    # divide by A'(k) = 1 - A^2 - (p-1)/k A, which cancels as Rbar -> 1
    # (A' ~ (p-1)/(2k^2)).  An error delta in A_p (relative) moves F by
    # [A + |step| (2A + (p-1)/k)] A delta / |A'|.  delta = difference of two
    # log I values, each computed with O(1) roundings of size eps |log I|:
    # delta = 2 * 32 eps max(|log I|, 1).
    eps = 2.0 ** -53

    def cond_tol(k_at, step, kref):
        A = ovmf.a_p(d, k_at)
        dA = abs(1 - A * A - (d - 1) / k_at * A)
        delta = 64 * eps * max(abs(float(oracle.log_iv(d / 2, k_at)[0])), 1.0)
        return 1e-12 * kref + (A + abs(step) * (2 * A + (d - 1) / k_at)) * A * delta / dA

    prev = ref["kappa0"]
    for i, k in ((2, "kappa1"), (3, "kappa2")):
        tol = cond_tol(prev, ref[k] - prev, ref[k])
        assert abs(s[i] - ref[k]) <= tol, (k, s[i], ref[k], tol)
        prev = ref[k]
    km = ref["kappa_mle"]
    tol = max(1e-9 * km, cond_tol(km, 0.0, km))
    assert abs(s[4] - km) <= tol, (s[4], km, tol)
    assert abs(s[5] - ref["loglik"]) <= 1e-10 * max(1, abs(ref["loglik"]))
    assert abs(s[6]) <= 1e-10                                   # stationarity A_p(k) = Rbar
    # Newton improvement ordering (Sra 2012; SPEC vmf property)
    r = ref["rbar"]
    g = [abs(ovmf.a_p(d, s[i]) - r) for i in (1, 2, 3)]
    assert g[2] <= g[1] * 1.0001 + 1e-15 and g[1] <= g[0] * 1.0001 + 1e-15


def test_table7_sufficient_statistics(B):
    """Paper Table 7 (lines 695-711): from Rbar = A_p(kappa2_paper) the device
    reproduces the printed kappa0/1/2 and the MLE equals kappa2 to ~1e-10."""
    import json, os
    rows = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "vmf_table7.json")))["rows"]
    for r in rows:
        p = r["p"]
        rbar = ovmf.a_p(p, r["kappa2"])
        colsum = torch.zeros(p, dtype=torch.float64, device="cuda:0")
        colsum[0] = rbar * 1000.0                              # n_total = 1000, xbar = rbar e_1
        mu, stats = B.vmf_fit_from_colsum(colsum, 1000)
        s = stats.cpu().numpy()
        tol = 1.5 * 10.0 ** (-r["digits"])
        assert abs(s[1] - r["kappa0"]) <= tol and abs(s[2] - r["kappa1"]) <= tol and abs(s[3] - r["kappa2"]) <= tol
        assert abs(s[4] - r["kappa2"]) / r["kappa2"] <= 1e-10


def test_degenerate(B):
    X = torch.tensor([[1.0, 0.0], [-1.0, 0.0]], dtype=torch.float64, device="cuda:0")
    _, stats = B.vmf_fit(X)
    s = stats.cpu().numpy()
    assert s[0] == 0.0 and np.all(np.isnan(s[1:]))


@pytest.mark.parametrize("d", [2048, 8192, 32768])
def test_full_size_features(B, d):
    """BASELINE configs[4]: 50000 x d unit-norm fp32 features (CIFAR10/ResNet50 shape)."""
    X, _ = workloads.vmf_features(50_000, d, rbar=0.17, seed=d, device="cuda:0", dtype=torch.float32)
    mu, stats = B.vmf_fit(X)
    s = stats.cpu().numpy()
    # sampled columns summed exactly on the host
    cols = np.random.default_rng(d).choice(d, 64, replace=False)
    Xc = X[:, torch.tensor(cols, device="cuda:0")].double().cpu().numpy()
    colsum = B.vmf_colsum(X).cpu().numpy()
    ref_cols = np.array([math.fsum(Xc[:, j]) for j in range(len(cols))])
    assert np.max(np.abs(colsum[cols] - ref_cols)) <= 1e-10
    rbar = ovmf.mean_resultant_rows(X.cpu().numpy())          # oracle input: the features only
    assert abs(s[0] - rbar) <= 1e-12
    k0, k1, k2 = ovmf.kappa_estimates(d, rbar)
    km = ovmf.kappa_mle(d, rbar)
    assert abs(s[3] - k2) <= 1e-9 * k2 and abs(s[4] - km) <= 1e-9 * km
    del X
    torch.cuda.empty_cache()


def test_colsum_concurrent_streams(B):
    """Column sums of two different matrices enqueued back to back on two streams with no
    synchronisation between them: each equals its single-stream result (the partials
    scratch is per (device, stream); include/bessel_b200.h thread-safety contract)."""
    Xa, _ = workloads.vmf_features(20_000, 2048, rbar=0.3, seed=5, device="cuda:0")
    Xb, _ = workloads.vmf_features(20_000, 2048, rbar=0.6, seed=6, device="cuda:0")
    ra = B.vmf_colsum(Xa).clone()
    rb = B.vmf_colsum(Xb).clone()
    torch.cuda.synchronize()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(5):
        with torch.cuda.stream(sa):
            ga = B.vmf_colsum(Xa)
        with torch.cuda.stream(sb):
            gb = B.vmf_colsum(Xb)
        with torch.cuda.stream(sa):
            ga2 = B.vmf_colsum(Xa)
        torch.cuda.synchronize()
        assert torch.equal(ga, ra) and torch.equal(gb, rb) and torch.equal(ga2, ra)


def test_with_count_layout_and_fit(B):
    """with_count: d column sums followed by the row count in one buffer (the single
    all-reduce of a sharded fit); vmf_fit_from_colsum(buf) reads n from the buffer and
    equals the fit with an explicit n_total.  accumulate adds both parts."""
    X, _ = workloads.vmf_features(3001, 256, rbar=0.4, seed=9, device="cuda:0", dtype=torch.float64)
    buf = B.vmf_colsum(X, with_count=True)
    assert buf.shape == (257,) and float(buf[256]) == 3001.0
    assert torch.equal(buf[:256], B.vmf_colsum(X))
    mu1, st1 = B.vmf_fit_from_colsum(buf)
    mu2, st2 = B.vmf_fit_from_colsum(buf[:256].clone(), 3001)
    assert torch.equal(mu1, mu2) and torch.equal(st1, st2)
    two = B.vmf_colsum(X, out=buf.clone(), accumulate=True, with_count=True)
    assert float(two[256]) == 6002.0 and torch.allclose(two[:256], 2 * buf[:256], rtol=1e-15, atol=0)
    mu3, st3 = B.vmf_fit(X)
    assert torch.equal(mu3, mu1) and torch.equal(st3, st1)
