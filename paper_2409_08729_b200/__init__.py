"""paper_2409_08729_b200 -- B200-native log I_v(x) / log K_v(x) and vMF fitting.

The hot path of arXiv 2409.08729: batched, log-scale evaluation of
the modified Bessel functions of the first and second kind, and the
von Mises-Fisher maximum-likelihood fit that consumes them.  Every step runs
in the sm_100a kernels of ``libbessel_b200.so`` (C ABI: include/bessel_b200.h);
this module only marshals torch CUDA tensors to device pointers and the
current CUDA stream.  There is no CPU fallback: calling with CPU tensors, or
without the built library, raises.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._build import build as build_library  # noqa: F401
from ._lib import B200Error, check, launch_count, lib  # noqa: F401

__all__ = [
    "log_iv", "log_kv", "log_ivkv", "log_kv_paper", "classify", "log_iv_host", "log_kv_host", "log_ivkv_host",
    "vmf_colsum", "vmf_fit_from_colsum", "vmf_fit", "VMF_STATS", "B200Error",
    "launch_count", "METHOD_MU", "METHOD_U13", "METHOD_FALLBACK",
]

METHOD_MU, METHOD_U13, METHOD_FALLBACK = 0, 1, 2
VMF_STATS = ("rbar", "kappa0", "kappa1", "kappa2", "kappa_mle", "loglik", "stationarity", "iterations")


def _stream(t: torch.Tensor):
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _pair(v: torch.Tensor, x: torch.Tensor, out):
    if not (isinstance(v, torch.Tensor) and isinstance(x, torch.Tensor)):
        raise TypeError("v and x must be torch tensors")
    if not (v.is_cuda and x.is_cuda):
        raise B200Error("inputs must be CUDA tensors (there is no CPU path)")
    if v.dtype != x.dtype or v.dtype not in (torch.float64, torch.float32):
        raise TypeError("v and x must share dtype float64 or float32")
    if v.shape != x.shape:
        raise ValueError("v and x must have the same shape")
    if v.device != x.device:
        raise ValueError("v and x must be on the same device")
    v = v.contiguous()
    x = x.contiguous()
    if out is None:
        out = torch.empty_like(v)
    elif out.shape != v.shape or out.dtype != v.dtype or out.device != v.device or not out.is_contiguous():
        raise ValueError("out must be a contiguous tensor like v")
    return v, x, out


def _call(name64, name32, v, x, out):
    v, x, out = _pair(v, x, out)
    fn = getattr(lib(), name64 if v.dtype == torch.float64 else name32)
    with torch.cuda.device(v.device):
        check(fn(v.data_ptr(), x.data_ptr(), out.data_ptr(), v.numel(), _stream(v)), fn.__name__)
    return out


def log_iv(v: torch.Tensor, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Elementwise log I_v(x) (§3.1, Algorithm 1); float64 or float32 CUDA tensors."""
    return _call("b200_log_iv_f64", "b200_log_iv_f32", v, x, out)


def log_kv(v: torch.Tensor, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Elementwise log K_v(x) (§3.2, Algorithm 1); float64 or float32 CUDA tensors."""
    return _call("b200_log_kv_f64", "b200_log_kv_f32", v, x, out)


def log_ivkv(v: torch.Tensor, x: torch.Tensor, out_i: torch.Tensor | None = None,
             out_k: torch.Tensor | None = None):
    """(log I_v(x), log K_v(x)) of the same pairs in one fused pass (shared loads, dispatch,
    and expansion terms); float64 or float32 CUDA tensors."""
    v, x, out_i = _pair(v, x, out_i)
    _, _, out_k = _pair(v, x, out_k)
    fn = lib().b200_log_ivkv_f64 if v.dtype == torch.float64 else lib().b200_log_ivkv_f32
    with torch.cuda.device(v.device):
        check(fn(v.data_ptr(), x.data_ptr(), out_i.data_ptr(), out_k.data_ptr(), v.numel(), _stream(v)),
              fn.__name__)
    return out_i, out_k


def log_kv_paper(v: torch.Tensor, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """log K_v(x) with the paper's own Simpson-integral fallback (float64 only)."""
    if v.dtype != torch.float64:
        raise TypeError("log_kv_paper is float64 only")
    return _call("b200_log_kv_paper_f64", "b200_log_kv_paper_f64", v, x, out)


def classify(v: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
    """Region id per element (METHOD_MU / METHOD_U13 / METHOD_FALLBACK; -1 invalid), int8."""
    if v.dtype != torch.float64:
        raise TypeError("classify takes float64 inputs")
    v, x, _ = _pair(v, x, None)
    m = torch.empty(v.shape, dtype=torch.int8, device=v.device)
    with torch.cuda.device(v.device):
        check(lib().b200_classify_f64(v.data_ptr(), x.data_ptr(), m.data_ptr(), v.numel(), _stream(v)),
              "b200_classify_f64")
    return m


def _host_arrays(v, x):
    """Host float64 inputs (CPU torch tensors or array-likes), contiguous, same shape."""
    if isinstance(v, torch.Tensor) or isinstance(x, torch.Tensor):
        if not (isinstance(v, torch.Tensor) and isinstance(x, torch.Tensor)):
            raise TypeError("host variants take two CPU tensors or two numpy arrays")
        if v.is_cuda or x.is_cuda or v.dtype != torch.float64 or x.dtype != torch.float64:
            raise TypeError("host variants take float64 CPU tensors or numpy arrays")
        v, x = v.contiguous(), x.contiguous()
    else:
        v = np.ascontiguousarray(v, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
    if tuple(v.shape) != tuple(x.shape):
        raise ValueError("v and x must have the same shape")
    return v, x


def _host_out(v, out):
    """A host float64 output like v (allocated if None; checked otherwise: the C call writes n doubles)."""
    if isinstance(v, torch.Tensor):
        if out is None:
            return torch.empty_like(v, pin_memory=v.is_pinned()), None
        if not isinstance(out, torch.Tensor) or out.is_cuda or out.dtype != torch.float64 \
                or tuple(out.shape) != tuple(v.shape) or not out.is_contiguous():
            raise ValueError("out must be a contiguous float64 CPU tensor shaped like v")
        return out, None
    if out is None:
        return np.empty_like(v), None
    if not isinstance(out, np.ndarray) or out.dtype != np.float64 or out.shape != v.shape \
            or not out.flags.c_contiguous or not out.flags.writeable:
        raise ValueError("out must be a writeable C-contiguous float64 numpy array shaped like v")
    return out, None


def _ptr(a):
    return a.data_ptr() if isinstance(a, torch.Tensor) else a.ctypes.data


def _host_call(name, v, x, out):
    v, x = _host_arrays(v, x)
    out, _ = _host_out(v, out)
    n = v.numel() if isinstance(v, torch.Tensor) else v.size
    check(getattr(lib(), name)(_ptr(v), _ptr(x), _ptr(out), n), name)
    return out


def log_iv_host(v, x, out=None):
    """log I_v(x) for HOST float64 arrays (pinned torch tensors or numpy); staged through the GPU."""
    return _host_call("b200_log_iv_f64_host", v, x, out)


def log_kv_host(v, x, out=None):
    """log K_v(x) for HOST float64 arrays (pinned torch tensors or numpy); staged through the GPU."""
    return _host_call("b200_log_kv_f64_host", v, x, out)


def log_ivkv_host(v, x, out_i=None, out_k=None):
    """(log I_v(x), log K_v(x)) for HOST float64 arrays in one fused pass: the inputs cross
    PCIe once for both functions."""
    v, x = _host_arrays(v, x)
    out_i, _ = _host_out(v, out_i)
    out_k, _ = _host_out(v, out_k)
    n = v.numel() if isinstance(v, torch.Tensor) else v.size
    check(lib().b200_log_ivkv_f64_host(_ptr(v), _ptr(x), _ptr(out_i), _ptr(out_k), n), "b200_log_ivkv_f64_host")
    return out_i, out_k


# ------------------------------------------------------------------ vMF
def _features(X: torch.Tensor):
    if not isinstance(X, torch.Tensor) or not X.is_cuda:
        raise B200Error("X must be a CUDA tensor (there is no CPU path)")
    if X.dim() != 2 or X.dtype not in (torch.float32, torch.float64):
        raise TypeError("X must be a 2-D float32/float64 tensor")
    if X.stride(1) != 1:
        X = X.contiguous()
    return X


def vmf_colsum(X: torch.Tensor, out: torch.Tensor | None = None, accumulate: bool = False,
               with_count: bool = False) -> torch.Tensor:
    """Column sums of the n x d features in float64 (the data-parallel part of the vMF fit).
    with_count: the result has d + 1 entries, the last one (+)= n (one all-reduce carries both)."""
    X = _features(X)
    n, d = X.shape
    m = d + 1 if with_count else d
    if out is None:
        out = torch.empty(m, dtype=torch.float64, device=X.device)
    elif (not isinstance(out, torch.Tensor) or not out.is_cuda or out.device != X.device
          or out.dtype != torch.float64 or out.shape != (m,) or not out.is_contiguous()):
        raise ValueError(f"out must be a contiguous float64 CUDA tensor of shape ({m},) on X's device")
    fn = lib().b200_vmf_colsum_f64 if X.dtype == torch.float64 else lib().b200_vmf_colsum_f32
    with torch.cuda.device(X.device):
        check(fn(X.data_ptr(), n, d, X.stride(0), out.data_ptr(), int(accumulate), int(with_count), _stream(X)),
              "vmf_colsum")
    return out


def vmf_fit_from_colsum(colsum: torch.Tensor, n_total: int | None = None):
    """mu (d,) and stats (8,) from the global column sum (§6.3).
    n_total None: colsum is a with_count sum of d + 1 entries whose last entry is the row count."""
    if not isinstance(colsum, torch.Tensor) or not colsum.is_cuda or colsum.dtype != torch.float64 \
            or colsum.dim() != 1:
        raise TypeError("colsum must be a 1-D float64 CUDA tensor")
    colsum = colsum.contiguous()
    d = colsum.numel() - (1 if n_total is None else 0)
    if n_total is not None and int(n_total) <= 0:
        raise ValueError("n_total must be positive")
    mu = torch.empty(d, dtype=torch.float64, device=colsum.device)
    stats = torch.empty(8, dtype=torch.float64, device=colsum.device)
    with torch.cuda.device(colsum.device):
        check(lib().b200_vmf_fit_from_colsum(colsum.data_ptr(), 0 if n_total is None else int(n_total), d,
                                             mu.data_ptr(), stats.data_ptr(), _stream(colsum)),
              "vmf_fit_from_colsum")
    return mu, stats


def vmf_fit(X: torch.Tensor, process_group=None):
    """Fit a vMF distribution to the rows of X (unit-norm features).

    With a torch.distributed process group the rows are a shard: the column
    sums and the row count travel in one buffer of d + 1 doubles and ONE
    all-reduce (NCCL on GPUs) sums them; every rank then computes the same fit
    on the device.  Returns (mu, stats) with stats named by VMF_STATS.
    """
    from .parallel import allreduce_colsum
    X = _features(X)
    buf = allreduce_colsum(vmf_colsum(X, with_count=True), process_group)
    return vmf_fit_from_colsum(buf)
