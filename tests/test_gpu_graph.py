"""CUDA-graph capture of the C-ABI calls (launch-bound small batches, serving loops).

The evaluation and vMF launches take device pointers and a stream and do no host
synchronisation, so a warmed-up call sequence can be captured once and replayed on new
inputs written into the same buffers.  The vMF column-sum scratch is per (device,
stream): the warm-up runs on the capture stream so the capture itself allocates nothing.
Replays must reproduce the direct calls bit for bit (the kernels are deterministic).
"""
import pytest
import torch

from paper_2409_08729_b200 import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2409_08729_b200 as B
    B.lib()
    return B


def test_capture_and_replay_fused_eval_and_vmf_fit(B):
    dev = torch.device("cuda:0")
    n = 3 * 2816 + 77                                  # several fused-pass tiles and a ragged tail
    v0, x0 = workloads.bench_grid(n // 11 + 1, seed=5, device=dev)
    v = v0[:n].contiguous()
    x = x0[:n].contiguous()
    X, _ = workloads.vmf_features(4000, 2048, rbar=0.2, seed=6, device=dev, dtype=torch.float32)
    oi = torch.empty_like(v)
    ok = torch.empty_like(v)
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):                         # warm-up on the capture stream
        B.log_ivkv(v, x, out_i=oi, out_k=ok)
        B.vmf_fit(X)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        B.log_ivkv(v, x, out_i=oi, out_k=ok)
        mu, stats = B.vmf_fit(X)
    for seed in (7, 8):
        v1, x1 = workloads.bench_grid(n // 11 + 1, seed=seed, device=dev)
        v.copy_(v1[:n].flip(0))
        x.copy_(x1[:n])
        X1, _ = workloads.vmf_features(4000, 2048, rbar=0.3, seed=seed, device=dev, dtype=torch.float32)
        X.copy_(X1)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        ri, rk = B.log_ivkv(v, x)
        rmu, rstats = B.vmf_fit(X)
        torch.cuda.synchronize()
        assert torch.equal(oi, ri) and torch.equal(ok, rk)
        assert torch.equal(mu, rmu) and torch.equal(stats, rstats)
