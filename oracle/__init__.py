"""oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously correct CPU references for the hot path of
arxiv 2409.08729 ("Robust and efficient computation of the logarithm of
modified Bessel functions"):

* ``log_iv`` / ``log_kv``  -- binary128 C (``bessel_oracle.c``): the series
  definition PAPER.md §3.1 Eq. (Iv infinite series) for I, and the integral
  representation DLMF 10.32.9 for K (see the C file's header for citations).
* ``vmf``                  -- the von Mises-Fisher estimators of PAPER.md §6.3
  (Eq. (mean direction estimate), Eq. (kappa estimates), the log-likelihood),
  in numpy float64 / math.fsum, calling ``log_iv`` above for A_p.

Who may import this package: ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs.  Nothing under
``paper_2409_08729_b200/`` imports it, and it imports nothing from there.

Parity status: every function here is pinned by ``tests/test_oracle_pins.py``
(closed forms, Wronskian, recurrences, mpmath/scipy library routines, the
paper's Table 7).  No function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bessel_oracle.c")
_LIB = os.path.join(_HERE, "libbessel_oracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the binary128 oracle with gcc (quadmath, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-o", _LIB, _SRC,
               "-lquadmath", "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            for name in ("oracle_log_iv", "oracle_log_kv",
                         "oracle_log_iv_serial", "oracle_log_kv_serial"):
                f = getattr(lib, name)
                f.restype = None
                f.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64]
            _lib = lib
    return _lib


def _call(name, v, x, with_lo=False):
    v = np.ascontiguousarray(np.broadcast_to(np.asarray(v, dtype=np.float64),
                                             np.broadcast_shapes(np.shape(v), np.shape(x))))
    x = np.ascontiguousarray(np.broadcast_to(np.asarray(x, dtype=np.float64), v.shape))
    hi = np.empty(v.shape, dtype=np.float64)
    lo = np.empty(v.shape, dtype=np.float64)
    n = v.size
    if n:
        getattr(_load(), name)(v.ctypes.data, x.ctypes.data, hi.ctypes.data, lo.ctypes.data, n)
    if hi.ndim == 0:
        hi, lo = float(hi), float(lo)
    if with_lo:
        return hi, lo
    return hi


def log_iv(v, x, with_lo: bool = False, serial: bool = False):
    """log I_v(x) for v >= 0, x >= 0 (binary128 series, rounded to float64).

    With ``with_lo`` returns (hi, lo) with hi + lo accurate to ~1e-32 relative.
    """
    return _call("oracle_log_iv_serial" if serial else "oracle_log_iv", v, x, with_lo)


def log_kv(v, x, with_lo: bool = False, serial: bool = False):
    """log K_v(x) for x > 0, any real v (binary128 integral, rounded to float64)."""
    return _call("oracle_log_kv_serial" if serial else "oracle_log_kv", v, x, with_lo)


def rel_err(got, ref):
    """Error measure used by every parity test (reading R1).

    |got - ref| / max(|ref|, 1): the relative error of the log value, floored
    at 1 because a log-domain result's absolute error equals the relative error
    of the function itself, so where log f crosses 0 a pure relative error is
    undefined.  Infinite values must match exactly.
    """
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    same_inf = np.isinf(got) & np.isinf(ref) & (np.sign(got) == np.sign(ref))
    with np.errstate(invalid="ignore"):
        e = np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)
    e = np.where(same_inf, 0.0, e)
    return np.where(np.isnan(e), np.inf, e)
