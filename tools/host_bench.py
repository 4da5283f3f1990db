"""Host-buffer pipeline variants (diagnostic): time b200_log_ivkv_f64_host of build/variants/*.so
on the e2e sample size (55M pairs from pinned host memory), wall clock, best of 3."""
import ctypes
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n = 55_000_000
g = torch.Generator().manual_seed(0)
v = (torch.randint(0, 11, (n,), generator=g).double().exp2()).pin_memory()
x = (torch.rand(n, generator=g, dtype=torch.float64) * 99 + 1).pin_memory()
oi = torch.empty(n, dtype=torch.float64).pin_memory()
ok = torch.empty(n, dtype=torch.float64).pin_memory()
torch.cuda.init()
res = {}
for nm in sys.argv[1:]:
    L = ctypes.CDLL(os.path.join(ROOT, "build", "variants", nm + ".so"))
    f = L.b200_log_ivkv_f64_host
    f.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64]
    f.restype = ctypes.c_int
    best = 1e9
    for _ in range(4):
        t = time.perf_counter()
        assert f(v.data_ptr(), x.data_ptr(), oi.data_ptr(), ok.data_ptr(), n) == 0
        best = min(best, time.perf_counter() - t)
    res[nm] = {"ms": round(best * 1e3, 2), "gevals": round(2 * n / best / 1e9, 3)}
print(json.dumps(res))
