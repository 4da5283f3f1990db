"""compute-sanitizer initcheck probe (diagnostic): does initcheck see bulk (TMA) stores?

Evaluates log I on 37 pairs twice -- once from 16-byte aligned tensors (results
leave shared memory through cp.async.bulk, one 288-byte bulk store + one plain
store for the tail element) and once from a view starting at element 1 (8-byte
aligned: plain per-thread stores only) -- and copies each result to the host.
Every output element is written by the kernel in both cases (the values are
checked against each other); an initcheck report on the first copy only means
the tool does not track writes made by the bulk-copy engine.
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2409_08729_b200 as B  # noqa: E402

dev = torch.device("cuda:0")
v = torch.linspace(0.5, 40.0, 38, dtype=torch.float64, device=dev)
x = torch.linspace(0.1, 90.0, 38, dtype=torch.float64, device=dev)
print("== aligned (bulk store)", flush=True)
a = B.log_iv(v[:37].clone(), x[:37].clone()).cpu()
torch.cuda.synchronize()
print("== unaligned view (plain stores)", flush=True)
b = B.log_iv(v[1:], x[1:]).cpu()
torch.cuda.synchronize()
ref = B.log_iv(v[1:].clone(), x[1:].clone()).cpu()
assert torch.equal(b, ref) and torch.isfinite(a).all(), "unexpected values"
print("probe ok", flush=True)
