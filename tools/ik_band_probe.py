import ctypes, os, sys, torch, json
sys.path.insert(0, os.getcwd())
import numpy as np, oracle
dev = torch.device("cuda:0")
n = 20_000_000
g = torch.Generator(device=dev).manual_seed(0)
x = torch.empty(n, dtype=torch.float32, device=dev).uniform_(1.0, 100.0, generator=g)
res = {}
outs = {}
for nm in ("old", "new"):
    L = ctypes.CDLL(f"build/variants/{nm}.so")
    f = L.b200_log_ivkv_f32
    f.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_void_p]
    s = torch.cuda.current_stream().cuda_stream
    tot = 0.0
    for j in range(11):
        v = torch.full((n,), float(2 ** j), dtype=torch.float32, device=dev)
        o1, o2 = torch.empty_like(v), torch.empty_like(v)
        f(v.data_ptr(), x.data_ptr(), o1.data_ptr(), o2.data_ptr(), n, s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            f(v.data_ptr(), x.data_ptr(), o1.data_ptr(), o2.data_ptr(), n, s)
        e1.record(); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1) / 5
    # band accuracy vs oracle (f32 inputs)
    rng = np.random.default_rng(5)
    vb = rng.uniform(0, 12.69, 20000).astype(np.float32); xb = rng.uniform(2.0, 30.0, 20000).astype(np.float32)
    vt, xt = torch.tensor(vb, device=dev), torch.tensor(xb, device=dev)
    o1, o2 = torch.empty_like(vt), torch.empty_like(vt)
    f(vt.data_ptr(), xt.data_ptr(), o1.data_ptr(), o2.data_ptr(), vb.size, s); torch.cuda.synchronize()
    ri = oracle.log_iv(vb.astype(np.float64), xb.astype(np.float64)); rk = oracle.log_kv(vb.astype(np.float64), xb.astype(np.float64))
    res[nm] = {"bench_grid_ms_f32": round(tot, 4), "band_err_i": float(oracle.rel_err(o1.double().cpu().numpy(), ri).max()),
               "band_err_k": float(oracle.rel_err(o2.double().cpu().numpy(), rk).max())}
    L64 = L.b200_log_ivkv_f64
    L64.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_void_p]
    vd, xd = vt.double(), xt.double()
    o1, o2 = torch.empty_like(vd), torch.empty_like(vd)
    L64(vd.data_ptr(), xd.data_ptr(), o1.data_ptr(), o2.data_ptr(), vb.size, s); torch.cuda.synchronize()
    res[nm]["band_err_i_f64"] = float(oracle.rel_err(o1.cpu().numpy(), ri).max())
    res[nm]["band_err_k_f64"] = float(oracle.rel_err(o2.cpu().numpy(), rk).max())
print(json.dumps(res))
