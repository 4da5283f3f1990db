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
X, _ = workloads.vmf_features(3000, 512, rbar=0.3, seed=1, device=dev)
B.vmf_fit(X)
B.vmf_fit(X.double())
torch.cuda.synchronize()
print("sanitize run ok")
