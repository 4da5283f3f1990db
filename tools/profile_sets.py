"""Run b200_log_ivkv_f64 of one library build once per method-homogeneous input set
(diagnostic driver for ncu; not the bench).

  ncu ... python tools/profile_sets.py build/variants/<name>.so u6 mu fb_b [--n N]
Sets as in tools/variant_bench.py (uniform boxes in (v, x)).
"""
import ctypes
import sys

import torch

BOXES = {
    "mu": ((0.0, 15.0), (30.0, 100.0)),
    "u6": ((512.0, 1024.0), (1.0, 100.0)),
    "u9": ((100.0, 256.0), (1.0, 60.0)),
    "u13": ((13.0, 60.0), (1.0, 40.0)),
    "fb_a": ((0.8, 12.0), (0.3, 2.0)),
    "fb_b": ((0.8, 12.0), (2.1, 19.0)),
    "grid1": ((1.0, 1.0), (1.0, 100.0)),
}


def main():
    lib = sys.argv[1]
    args = sys.argv[2:]
    names = [a for i, a in enumerate(args) if not a.startswith("--") and not (i and args[i - 1] == "--n")]
    n = int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 4_000_000
    L = ctypes.CDLL(lib)
    L.b200_log_ivkv_f64.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_void_p]
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    s = torch.cuda.current_stream(dev).cuda_stream
    for nm in names:
        (v0, v1), (x0, x1) = BOXES[nm]
        v = torch.empty(n, dtype=torch.float64, device=dev).uniform_(v0, v1, generator=g)
        x = torch.empty(n, dtype=torch.float64, device=dev).uniform_(x0, x1, generator=g)
        o1, o2 = torch.empty_like(v), torch.empty_like(v)
        rc = L.b200_log_ivkv_f64(v.data_ptr(), x.data_ptr(), o1.data_ptr(), o2.data_ptr(), n, s)
        torch.cuda.synchronize()
        print(nm, rc, flush=True)


if __name__ == "__main__":
    main()
