"""Small-batch latency: direct C-ABI calls vs one CUDA graph replaying many calls (diagnostic).

A serving loop evaluates many small batches; each b200_log_ivkv_f64 launch then costs
its launch overhead more than its work.  Capturing CALLS calls into one graph and
replaying it removes the per-call host overhead.  Prints one JSON line per batch size.
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2409_08729_b200 as B  # noqa: E402
from paper_2409_08729_b200 import workloads  # noqa: E402

CALLS = 100


def main():
    dev = torch.device("cuda:0")
    s = torch.cuda.Stream(dev)
    for n in (1536, 15360, 153600, 1536000):
        v0, x0 = workloads.bench_grid(n // 11 + 1, seed=1, device=dev)
        v, x = v0[:n].contiguous(), x0[:n].contiguous()
        oi, ok = torch.empty_like(v), torch.empty_like(v)
        with torch.cuda.stream(s):
            for _ in range(3):
                B.log_ivkv(v, x, out_i=oi, out_k=ok)
            s.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(CALLS):
                B.log_ivkv(v, x, out_i=oi, out_k=ok)
            e1.record(s)
            e1.synchronize()
            direct = e0.elapsed_time(e1) / CALLS
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(CALLS):
                B.log_ivkv(v, x, out_i=oi, out_k=ok)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            g.replay()
            e1.record(s)
        e1.synchronize()
        graph = e0.elapsed_time(e1) / CALLS
        print(json.dumps({"pairs_per_call": n, "direct_us_per_call": round(1e3 * direct, 2),
                          "graph_us_per_call": round(1e3 * graph, 2),
                          "direct_gevals": round(2 * n / direct / 1e6, 2),
                          "graph_gevals": round(2 * n / graph / 1e6, 2)}), flush=True)


if __name__ == "__main__":
    main()
