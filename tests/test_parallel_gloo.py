"""Multi-process (world_size 2, gloo, CPU) checks of the sharding / all-reduce host logic."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_08729_b200.parallel import allreduce_colsum, shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 220_000_000, 50_000):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, X, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(X.shape[0], world, rank)
    # stand-in for b200_vmf_colsum_* with with_count: [column sums..., row count]
    buf = torch.tensor(np.concatenate([X[lo:hi].sum(axis=0), [hi - lo]]), dtype=torch.float64)
    calls = []
    real = dist.all_reduce

    def counting(*a, **k):
        calls.append(1)
        return real(*a, **k)
    dist.all_reduce = counting
    try:
        out = allreduce_colsum(buf)
    finally:
        dist.all_reduce = real
    q.put((rank, out.numpy(), len(calls)))
    dist.barrier()
    dist.destroy_process_group()


def test_allreduce_colsum_world2():
    """The sharded vMF fit's only exchange: ONE all-reduce of d + 1 doubles (column sums
    and the row count), identical on every rank."""
    rng = np.random.default_rng(0)
    X = rng.normal(size=(1001, 37))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, X, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    full = X.sum(axis=0)
    for rank, buf, ncalls in res:
        assert ncalls == 1
        assert buf[-1] == 1001
        assert np.allclose(buf[:-1], full, rtol=1e-13, atol=1e-12)
    assert np.array_equal(res[0][1], res[1][1])   # every rank sees the same reduced vector


def test_allreduce_colsum_single_process_is_identity():
    buf = torch.arange(5, dtype=torch.float64)
    assert allreduce_colsum(buf) is buf


def _fit_worker(rank, world, port, X, q):
    """vmf_fit(process_group=...) on a row shard, with the two device calls replaced by CPU
    stand-ins (no GPU here): the composition issues exactly one all-reduce, of d + 1 doubles."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2409_08729_b200 as B
    B._features = lambda X: X
    B.vmf_colsum = lambda X, with_count=False: torch.cat(
        [X.sum(0, dtype=torch.float64), torch.tensor([float(X.shape[0])], dtype=torch.float64)])
    B.vmf_fit_from_colsum = lambda buf: (buf[:-1] / buf[-1], buf)
    sizes = []
    real = dist.all_reduce

    def counting(t, *a, **k):
        sizes.append(t.numel())
        return real(t, *a, **k)
    dist.all_reduce = counting
    lo, hi = shard_range(X.shape[0], world, rank)
    try:
        xbar, buf = B.vmf_fit(torch.tensor(X[lo:hi]), process_group=dist.group.WORLD)
    finally:
        dist.all_reduce = real
    q.put((rank, sizes, xbar.numpy(), float(buf[-1])))
    dist.barrier()
    dist.destroy_process_group()


def test_vmf_fit_process_group_one_collective():
    rng = np.random.default_rng(1)
    X = rng.normal(size=(777, 19))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fit_worker, args=(r, 2, port, X, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, sizes, xbar, n in res:
        assert sizes == [19 + 1]
        assert n == 777
        assert np.allclose(xbar, X.mean(axis=0), rtol=1e-13, atol=1e-15)


def test_vmf_features_shards_are_slices_of_one_matrix():
    """bench.py's sharded vMF leg: rank r's rows are rows shard_range(n, N, r) of the one
    matrix the N = 1 run fits (mu and rows independent of the world size)."""
    from paper_2409_08729_b200 import workloads
    X, mu = workloads.vmf_features(1000, 64, rbar=0.3, seed=5, device="cpu")
    for w in (2, 3, 8):
        parts = [workloads.vmf_features(1000, 64, rbar=0.3, seed=5, device="cpu",
                                        rows=shard_range(1000, w, r)) for r in range(w)]
        assert torch.equal(torch.cat([p[0] for p in parts]), X)
        assert all(torch.equal(p[1], mu) for p in parts)


def test_bench_grid_slices_are_slices_of_one_grid():
    """bench.py's strong-scaling leg: the shards of every world size tile one global grid."""
    from paper_2409_08729_b200 import workloads
    v, x = workloads.bench_grid_slice(1000, 0, 11000, device="cpu")
    assert torch.equal(v[::1000], torch.tensor(workloads.BENCH_ORDERS, dtype=torch.float64))
    for w in (2, 3, 8):
        parts = [workloads.bench_grid_slice(1000, *shard_range(11000, w, r), device="cpu") for r in range(w)]
        assert torch.equal(torch.cat([p[0] for p in parts]), v)
        assert torch.equal(torch.cat([p[1] for p in parts]), x)
