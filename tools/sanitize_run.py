"""Small invocations of every kernel for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2409_08729_b200 as B  # noqa: E402
from paper_2409_08729_b200 import workloads  # noqa: E402

dev = torch.device("cuda:0")
rng = np.random.default_rng(0)
for n in (1, 37, 1024, 3001, 70000):
    v = np.exp(rng.uniform(np.log(1e-3), np.log(2e3), n))
    x = np.exp(rng.uniform(np.log(1e-3), np.log(2e3), n))
    v[:3] = [0.0, -1.0, np.nan][:min(3, n)] if n >= 3 else v[:n]
    for dt in (torch.float64, torch.float32):
        vt, xt = torch.tensor(v, dtype=dt, device=dev), torch.tensor(x, dtype=dt, device=dev)
        B.log_iv(vt, xt)
        B.log_kv(vt, xt)
        B.log_ivkv(vt, xt)
        B.log_iv(vt[1:], xt[1:])          # unaligned -> cp.async path
        B.log_ivkv(vt[1:], xt[1:])
    B.log_kv_paper(torch.tensor(v, device=dev), torch.tensor(x, device=dev))
    B.classify(torch.tensor(np.abs(v), device=dev), torch.tensor(x, device=dev))
    B.log_ivkv_host(np.abs(v), x)
# single-bin tiles (the homogeneous path that skips the sort and one barrier) mixed
# with sorted tiles in one launch: v = 512 (U6) then v = 1 (mu / U13 / fallback)
for dt in (torch.float64, torch.float32):
    vh = torch.cat([torch.full((5000,), 512.0), torch.full((3000,), 1.0)]).to(dt).to(dev)
    xh = torch.linspace(1.0, 100.0, 8000, dtype=dt, device=dev)
    B.log_ivkv(vh, xh)
    B.log_iv(vh, xh)
    B.log_kv(vh, xh)
# tiny and huge arguments (the slow bin)
vt = torch.tensor([0.0, 0.3, 5.5, 12.6, 100.0, 1e150, 2.0], device=dev)
xt = torch.tensor([5e-324, 1e-310, 1e-200, 1e-150, 1e300, 3.0, 1e200], device=dev)
B.log_ivkv(vt, xt)
X, _ = workloads.vmf_features(3000, 512, rbar=0.3, seed=1, device=dev)
B.vmf_fit(X)
B.vmf_fit(X.double())
B.vmf_colsum(X, with_count=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
with torch.cuda.stream(s1):
    B.vmf_colsum(X)
with torch.cuda.stream(s2):
    B.vmf_colsum(X.double())
torch.cuda.synchronize()
print("sanitize run ok")
