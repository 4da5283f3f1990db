"""Wide-domain accuracy probe (diagnostic, GPU box): 2M log-uniform pairs v, x in [1e-3, 1e5]
per precision, all three entry points against the binary128 oracle (profiles/r170)."""
import sys, json
import numpy as np, torch
sys.path.insert(0, ".")
import oracle
import paper_2409_08729_b200 as B
rng = np.random.default_rng(17)
n = 2_000_000
out = {}
for dt, name in ((torch.float32, "f32"), (torch.float64, "f64")):
    v = np.exp(rng.uniform(np.log(1e-3), np.log(1e5), n)); x = np.exp(rng.uniform(np.log(1e-3), np.log(1e5), n))
    if dt == torch.float32:
        v = v.astype(np.float32).astype(np.float64); x = x.astype(np.float32).astype(np.float64)
    vt = torch.tensor(v, device="cuda:0", dtype=dt); xt = torch.tensor(x, device="cuda:0", dtype=dt)
    ri, rk = oracle.log_iv(v, x), oracle.log_kv(v, x)
    fi, fk = B.log_ivkv(vt, xt)
    row = {}
    for what, got, ref in (("iv", B.log_iv(vt, xt), ri), ("kv", B.log_kv(vt, xt), rk), ("ivkv_i", fi, ri), ("ivkv_k", fk, rk)):
        g = got.double().cpu().numpy()
        e = oracle.rel_err(g, ref); i = int(np.argmax(e))
        row[what] = {"max": float(e[i]), "at": [float(v[i]), float(x[i])], "nonfinite": int((~np.isfinite(g)).sum())}
    out[name] = row
    print(name, row, flush=True)
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "wide.json", "w"), indent=1)
