"""Pinned host <-> device copy bandwidth on the box (diagnostic): the ceiling of bench.py's e2e.

Copies the e2e sample's bytes (55M pairs: 880 MB each way) H2D and D2H, alone
and concurrently on two streams, and prints GB/s per direction.
"""
import json
import time

import torch

n = 110_000_000                                  # doubles: 55M pairs x (v, x) = 880 MB
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for mode in ("h2d", "d2h", "both", "h2d", "d2h", "both"):
    torch.cuda.synchronize()
    t = time.perf_counter()
    if mode in ("h2d", "both"):
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
    if mode in ("d2h", "both"):
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    res[mode] = round(n * 8 / dt / 1e9, 1)
print(json.dumps({"GB_per_s_per_direction": res, "bytes_each_way": n * 8}))
