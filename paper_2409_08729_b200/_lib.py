"""ctypes binding of include/bessel_b200.h (argument marshalling only)."""
from __future__ import annotations

import ctypes
import os
import threading

from ._build import LIB

_lock = threading.Lock()
_lib = None

P = ctypes.c_void_p
I64 = ctypes.c_int64
INT = ctypes.c_int

SIGNATURES = {
    "b200_log_iv_f64": [P, P, P, I64, P],
    "b200_log_iv_f32": [P, P, P, I64, P],
    "b200_log_kv_f64": [P, P, P, I64, P],
    "b200_log_kv_f32": [P, P, P, I64, P],
    "b200_log_kv_paper_f64": [P, P, P, I64, P],
    "b200_log_ivkv_f64": [P, P, P, P, I64, P],
    "b200_log_ivkv_f32": [P, P, P, P, I64, P],
    "b200_classify_f64": [P, P, P, I64, P],
    "b200_log_iv_f64_host": [P, P, P, I64],
    "b200_log_kv_f64_host": [P, P, P, I64],
    "b200_log_ivkv_f64_host": [P, P, P, P, I64],
    "b200_vmf_colsum_f32": [P, I64, I64, I64, P, INT, INT, P],
    "b200_vmf_colsum_f64": [P, I64, I64, I64, P, INT, INT, P],
    "b200_vmf_fit_from_colsum": [P, I64, I64, P, P, P],
    "b200_vmf_fit_f32": [P, I64, I64, P, P, P, P],
    "b200_vmf_fit_f64": [P, I64, I64, P, P, P, P],
    "b200_last_error": [],
    "b200_launch_count": [],
}


class B200Error(RuntimeError):
    pass


def lib():
    """Load libbessel_b200.so; raise if it has not been built (no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB):
                raise B200Error(
                    f"{LIB} is missing: run __graft_entry__.build() or "
                    "`python -m paper_2409_08729_b200._build` (there is no CPU fallback)")
            L = ctypes.CDLL(LIB)
            for name, args in SIGNATURES.items():
                f = getattr(L, name)
                f.argtypes = args
                f.restype = INT
            L.b200_last_error.restype = ctypes.c_char_p
            L.b200_launch_count.restype = I64
            _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().b200_last_error().decode(errors="replace")
        raise B200Error(f"{what} failed (status {rc}): {msg}")


def launch_count() -> int:
    return int(lib().b200_launch_count())
