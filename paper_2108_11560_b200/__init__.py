"""B200-native (sm_100a) batched log K_v(x), d/dv and d/dx by Takekawa's
fixed-bin integral method (arXiv 2108.11560).

Thin ctypes binding over ``libbessel_logk.so`` (C ABI in
``include/bessel_logk.h``).  Argument marshalling only: every step of the
method runs in the CUDA kernels.  PyTorch provides device memory and streams.
There is no CPU fallback: if the shared library is missing the import of the
native handle raises.

    import torch, paper_2108_11560_b200 as blk
    v = torch.rand(1 << 20, dtype=torch.float64, device="cuda") * 100
    x = torch.rand(1 << 20, dtype=torch.float64, device="cuda") * 10 + 0.1
    logk, dv, dx = blk.log_bessel_k(v, x, nbins=128)
"""
from __future__ import annotations

import ctypes
import os
import re

__all__ = [
    "BLK_OK", "BLK_EINVAL", "BLK_ECUDA", "BLK_RANGE_AUTO", "BLK_RANGE_F64",
    "BLK_KERNEL_AUTO", "BLK_KERNEL_SIMPLE", "BLK_KERNEL_VEC128",
    "BesselLogKError", "lib", "library_path", "header_functions",
    "bessel_logk_f64", "bessel_logk_f32", "log_bessel_k", "bessel_logk_f64_host",
    "bessel_logk_f32_host",
    "host_workspace_bytes", "microbench", "DEFAULT_NBINS", "nig_loglik", "log_bessel_k_hess",
    "bessel_logk_plan_f64",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
library_path = os.path.join(_HERE, "libbessel_logk.so")
HEADER = os.path.join(_ROOT, "include", "bessel_logk.h")

BLK_OK, BLK_EINVAL, BLK_ECUDA = 0, 1, 2
BLK_RANGE_AUTO, BLK_RANGE_F64 = 0, 1
BLK_KERNEL_AUTO, BLK_KERNEL_SIMPLE, BLK_KERNEL_VEC128 = 0, 1, 2
BLK_MB_UNROLL = 16
# Trapezoid intervals used when the caller gives none (the paper states no n,
# P:222; R10).
DEFAULT_NBINS = 128


class BesselLogKError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"bessel_logk status {status}: {msg}")
        self.status = status


class _Options(ctypes.Structure):
    _fields_ = [("lanes_per_element", ctypes.c_int), ("range_mode", ctypes.c_int),
                ("block_threads", ctypes.c_int), ("kernel", ctypes.c_int)]


_lib = None


def lib():
    """The loaded native library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(library_path):
            raise ImportError(
                f"{library_path} not found: build it with "
                "`python -m paper_2108_11560_b200.build` (no CPU fallback exists)")
        L = ctypes.CDLL(library_path)
        vp, sz, ci = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
        for name in ("bessel_logk_f64", "bessel_logk_f32"):
            f = getattr(L, name)
            f.restype = ci
            f.argtypes = [vp, vp, sz, vp, vp, vp, ci, vp]
        for name in ("bessel_logk_f64_ex", "bessel_logk_f32_ex"):
            f = getattr(L, name)
            f.restype = ci
            f.argtypes = [vp, vp, sz, vp, vp, vp, ci, ctypes.POINTER(_Options), vp]
        L.bessel_logk_host_workspace_bytes.restype = sz
        L.bessel_logk_host_workspace_bytes.argtypes = [sz, sz]
        for name in ("bessel_logk_f64_host", "bessel_logk_f32_host"):
            f = getattr(L, name)
            f.restype = ci
            f.argtypes = [vp, vp, sz, vp, vp, vp, ci, vp, sz, sz, vp]
        L.bessel_logk_last_error.restype = ctypes.c_char_p
        L.bessel_logk_version.restype = ctypes.c_char_p
        L.bessel_logk_hess_f64.restype = ci
        L.bessel_logk_hess_f64.argtypes = [vp, vp, sz, vp, vp, vp, vp, vp, vp, ci,
                                           ctypes.POINTER(_Options), vp]
        L.bessel_logk_plan_f64.restype = ci
        L.bessel_logk_plan_f64.argtypes = [vp, vp, sz, vp, vp, vp, vp, ci,
                                           ctypes.POINTER(_Options), vp]
        L.bessel_nig_workspace_bytes.restype = sz
        L.bessel_nig_workspace_bytes.argtypes = [sz]
        cd = ctypes.c_double
        L.bessel_nig_loglik_f64.restype = ci
        L.bessel_nig_loglik_f64.argtypes = [vp, sz, cd, cd, cd, cd, ci, vp, vp, sz, vp]
        for name in ("blk_microbench_fp64", "blk_microbench_fp32", "blk_microbench_mufu"):
            f = getattr(L, name)
            f.restype = ci
            f.argtypes = [ci, ci, ci, vp, vp]
        _lib = L
    return _lib


def header_functions():
    """Names of every function declared in include/bessel_logk.h."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"BLK_API\s+[\w\s\*]+?\b(\w+)\s*\(", txt)))


def _check(st):
    if st != BLK_OK:
        raise BesselLogKError(st, lib().bessel_logk_last_error().decode())


def _stream_for(stream, device):
    """The stream to enqueue on (the device's current stream when None); it
    must belong to ``device`` (a foreign stream handle would launch on
    another GPU's pointers)."""
    import torch
    if stream is None:
        return torch.cuda.current_stream(device)
    if stream.device != device:
        raise ValueError(f"stream is on {stream.device}, tensors on {device}")
    return stream


def _stream_handle(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _keep_alive(stream, *tensors):
    """Tensors allocated here (outputs, temporaries, workspaces) come from the
    caching allocator on the CURRENT stream; when the kernel runs on another
    stream, record that use so their memory is not reused before it ends."""
    import torch
    if stream != torch.cuda.current_stream(stream.device):
        for t in tensors:
            if t is not None:
                t.record_stream(stream)


def _dev_ptr(t, dtype, n, name, device=None):
    import torch
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device} (all tensors on one GPU)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous() or t.numel() != n:
        raise ValueError(f"{name} must be contiguous with {n} elements")
    return ctypes.c_void_p(t.data_ptr())


def _opts(lanes_per_element, range_mode, block_threads, kernel):
    if lanes_per_element == 0 and range_mode == 0 and block_threads == 0 and kernel == 0:
        return None
    return _Options(int(lanes_per_element), int(range_mode), int(block_threads), int(kernel))


def _call(prec, v, x, logk, dlogk_dv, dlogk_dx, nbins, stream, lanes_per_element,
          range_mode, block_threads, kernel):
    import torch
    dtype = torch.float64 if prec == 64 else torch.float32
    if not isinstance(v, torch.Tensor) or not v.is_cuda:
        raise TypeError("v must be a CUDA tensor")
    dev = v.device
    n = v.numel()
    pv = _dev_ptr(v, dtype, n, "v", dev)
    px = _dev_ptr(x, dtype, n, "x", dev)
    po = [_dev_ptr(t, dtype, n, nm, dev) for t, nm in
          ((logk, "logk"), (dlogk_dv, "dlogk_dv"), (dlogk_dx, "dlogk_dx"))]
    L = lib()
    o = _opts(lanes_per_element, range_mode, block_threads, kernel)
    st = _stream_for(stream, dev)
    s = ctypes.c_void_p(st.cuda_stream)
    with torch.cuda.device(dev):
        if o is None:
            f = L.bessel_logk_f64 if prec == 64 else L.bessel_logk_f32
            _check(f(pv, px, n, po[0], po[1], po[2], int(nbins), s))
        else:
            f = L.bessel_logk_f64_ex if prec == 64 else L.bessel_logk_f32_ex
            _check(f(pv, px, n, po[0], po[1], po[2], int(nbins), ctypes.byref(o), s))
    return st


def bessel_logk_f64(v, x, logk=None, dlogk_dv=None, dlogk_dx=None, nbins=DEFAULT_NBINS,
                    stream=None, lanes_per_element=0, range_mode=BLK_RANGE_AUTO,
                    block_threads=0, kernel=BLK_KERNEL_AUTO):
    """Enqueue the FP64 kernel on ``stream`` writing into the given float64 CUDA tensors."""
    _call(64, v, x, logk, dlogk_dv, dlogk_dx, nbins, stream, lanes_per_element,
          range_mode, block_threads, kernel)


def bessel_logk_f32(v, x, logk=None, dlogk_dv=None, dlogk_dx=None, nbins=DEFAULT_NBINS,
                    stream=None, lanes_per_element=0, range_mode=BLK_RANGE_AUTO,
                    block_threads=0, kernel=BLK_KERNEL_AUTO):
    """Enqueue the FP32 kernel on ``stream`` writing into the given float32 CUDA tensors."""
    _call(32, v, x, logk, dlogk_dv, dlogk_dx, nbins, stream, lanes_per_element,
          range_mode, block_threads, kernel)


def log_bessel_k(v, x, nbins=DEFAULT_NBINS, outputs=("logk", "dv", "dx"), **kw):
    """Allocate outputs and evaluate; returns a tuple in the order of ``outputs``."""
    import torch
    dt = v.dtype
    if dt not in (torch.float64, torch.float32):
        raise TypeError("v must be float64 or float32")
    want = {k: (torch.empty_like(v) if k in outputs else None) for k in ("logk", "dv", "dx")}
    xc = x.to(dt).contiguous()
    st = _call(64 if dt == torch.float64 else 32, v, xc, want["logk"], want["dv"], want["dx"],
               nbins, kw.pop("stream", None), kw.pop("lanes_per_element", 0),
               kw.pop("range_mode", BLK_RANGE_AUTO), kw.pop("block_threads", 0),
               kw.pop("kernel", BLK_KERNEL_AUTO))
    if kw:
        raise TypeError(f"unexpected arguments {sorted(kw)}")
    _keep_alive(st, xc if xc is not x else None, *want.values())
    return tuple(want[k] for k in outputs)


def host_workspace_bytes(chunk=0, elem_bytes=8):
    return lib().bessel_logk_host_workspace_bytes(int(chunk), int(elem_bytes))


def _host_call(prec, v, x, logk, dlogk_dv, dlogk_dx, nbins, workspace, chunk, stream):
    import torch
    dtype = torch.float64 if prec == 64 else torch.float32
    n = v.numel()

    def hp(t, name):
        if t is None:
            return None
        if t.is_cuda or t.dtype != dtype or not t.is_contiguous() or t.numel() != n:
            raise TypeError(f"{name} must be a contiguous CPU {dtype} tensor of {n} elements")
        return ctypes.c_void_p(t.data_ptr())

    if workspace is not None and not workspace.is_cuda:
        raise TypeError("workspace must be a CUDA tensor (or None on the zero-copy transport)")
    dev = workspace.device if workspace is not None else (
        stream.device if stream is not None else torch.device("cuda", torch.cuda.current_device()))
    st = _stream_for(stream, dev)
    f = lib().bessel_logk_f64_host if prec == 64 else lib().bessel_logk_f32_host
    wp = ctypes.c_void_p(workspace.data_ptr()) if workspace is not None else None
    wb = workspace.numel() * workspace.element_size() if workspace is not None else 0
    with torch.cuda.device(dev):
        _check(f(hp(v, "v"), hp(x, "x"), n, hp(logk, "logk"), hp(dlogk_dv, "dlogk_dv"),
                 hp(dlogk_dx, "dlogk_dx"), int(nbins), wp, wb, int(chunk),
                 ctypes.c_void_p(st.cuda_stream)))


def bessel_logk_f64_host(v, x, logk=None, dlogk_dv=None, dlogk_dx=None, nbins=DEFAULT_NBINS,
                         workspace=None, chunk=0, stream=None):
    """Host-buffer entry point: v, x, outputs are CPU float64 tensors.  All pinned
    (torch pin_memory): zero-copy, ``workspace`` may be None.  Otherwise (staged
    transport) ``workspace`` is a CUDA uint8 tensor of >= host_workspace_bytes(chunk)
    bytes.  Blocking: returns with the results in the host tensors."""
    _host_call(64, v, x, logk, dlogk_dv, dlogk_dx, nbins, workspace, chunk, stream)


def bessel_logk_f32_host(v, x, logk=None, dlogk_dv=None, dlogk_dx=None, nbins=DEFAULT_NBINS,
                         workspace=None, chunk=0, stream=None):
    """FP32 host-buffer entry point: CPU float32 tensors; ``workspace`` of >=
    host_workspace_bytes(chunk, 4) bytes."""
    _host_call(32, v, x, logk, dlogk_dv, dlogk_dx, nbins, workspace, chunk, stream)


def microbench(kind, blocks, threads, iters, out, stream=None):
    """Enqueue a peak-rate microbenchmark ('fp64' DFMA, 'fp32' FFMA, 'mufu' EX2).
    Returns the instruction count it executes."""
    f = {"fp64": lib().blk_microbench_fp64, "fp32": lib().blk_microbench_fp32,
         "mufu": lib().blk_microbench_mufu}[kind]
    _check(f(int(blocks), int(threads), int(iters), ctypes.c_void_p(out.data_ptr()),
             _stream_handle(stream)))
    return blocks * threads * iters * BLK_MB_UNROLL


def nig_loglik(y, alpha, beta, delta, mu, nbins=DEFAULT_NBINS, out=None, workspace=None,
               stream=None):
    """Sum of NIG log-densities of the float64 CUDA tensor ``y`` and its gradient in
    (alpha, beta, delta, mu): returns a CUDA float64 tensor of 5 values (one device pass,
    no host sync).  See include/bessel_logk.h (bessel_nig_loglik_f64)."""
    import torch
    if not isinstance(y, torch.Tensor) or not y.is_cuda:
        raise TypeError("y must be a CUDA tensor")
    dev = y.device
    n = y.numel()
    py = _dev_ptr(y, torch.float64, n, "y", dev)
    st = _stream_for(stream, dev)
    made = []
    if out is None:
        out = torch.empty(5, dtype=torch.float64, device=dev)
        made.append(out)
    _dev_ptr(out, torch.float64, 5, "out", dev)
    nbytes = lib().bessel_nig_workspace_bytes(n)
    if workspace is None or workspace.numel() * workspace.element_size() < nbytes:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        made.append(workspace)
    elif workspace.device != dev:
        raise ValueError(f"workspace is on {workspace.device}, expected {dev}")
    with torch.cuda.device(dev):
        _check(lib().bessel_nig_loglik_f64(
            py, n, float(alpha), float(beta), float(delta), float(mu), int(nbins),
            ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(workspace.data_ptr()),
            workspace.numel() * workspace.element_size(), ctypes.c_void_p(st.cuda_stream)))
    _keep_alive(st, *made)
    return out


def log_bessel_k_hess(v, x, nbins=DEFAULT_NBINS, stream=None, lanes_per_element=0,
                      range_mode=BLK_RANGE_AUTO):
    """(log K, dv, dx, d2/dv2, d2/dx2, d2/dvdx) of float64 CUDA tensors in one pass."""
    import torch
    if not isinstance(v, torch.Tensor) or not v.is_cuda:
        raise TypeError("v must be a CUDA tensor")
    dev = v.device
    n = v.numel()
    pv = _dev_ptr(v, torch.float64, n, "v", dev)
    px = _dev_ptr(x, torch.float64, n, "x", dev)
    st = _stream_for(stream, dev)
    outs = [torch.empty_like(v) for _ in range(6)]
    o = _Options(int(lanes_per_element), int(range_mode), 0, 0)
    with torch.cuda.device(dev):
        _check(lib().bessel_logk_hess_f64(pv, px, n, *[ctypes.c_void_p(t.data_ptr()) for t in outs],
                                          int(nbins), ctypes.byref(o),
                                          ctypes.c_void_p(st.cuda_stream)))
    _keep_alive(st, *outs)
    return tuple(outs)


def bessel_logk_plan_f64(v, x, nbins=DEFAULT_NBINS, stream=None, range_mode=BLK_RANGE_AUTO):
    """The integration plan (t_p, g(t_p), t0, t1) the FP64 entry point integrates
    over for this nbins and range_mode, as four float64 CUDA tensors (NaN where an
    element has none).  See include/bessel_logk.h (bessel_logk_plan_f64)."""
    import torch
    if not isinstance(v, torch.Tensor) or not v.is_cuda:
        raise TypeError("v must be a CUDA tensor")
    dev = v.device
    n = v.numel()
    pv = _dev_ptr(v, torch.float64, n, "v", dev)
    px = _dev_ptr(x, torch.float64, n, "x", dev)
    st = _stream_for(stream, dev)
    outs = [torch.empty_like(v) for _ in range(4)]
    o = _Options(0, int(range_mode), 0, 0)
    with torch.cuda.device(dev):
        _check(lib().bessel_logk_plan_f64(pv, px, n, *[ctypes.c_void_p(t.data_ptr()) for t in outs],
                                          int(nbins), ctypes.byref(o),
                                          ctypes.c_void_p(st.cuda_stream)))
    _keep_alive(st, *outs)
    return tuple(outs)
