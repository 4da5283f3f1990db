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
    part = torch.tensor(X[lo:hi].sum(axis=0), dtype=torch.float64)   # stand-in for b200_vmf_colsum
    colsum, n = allreduce_colsum(part, hi - lo)
    q.put((rank, colsum.numpy(), n))
    dist.barrier()
    dist.destroy_process_group()


def test_allreduce_colsum_world2():
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
    for rank, cs, n in res:
        assert n == 1001
        assert np.allclose(cs, full, rtol=1e-13, atol=1e-12)
    assert np.array_equal(res[0][1], res[1][1])   # every rank sees the same reduced vector
