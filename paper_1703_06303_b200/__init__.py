"""B200 (sm_100a) implementation of the per-iteration sWLR update of Dutta & Li,
"A Fast Algorithm for a Weighted Low Rank Approximation" (arXiv 1703.06303).

The functions below carry the names of the C ABI in ``include/wlr.h`` and only marshal
arguments; all arithmetic runs in ``libwlr.so``.  Arrays may be torch CUDA tensors
(device pointers, BORROWED by the handle: keep them alive) or numpy arrays / CPU
tensors (host pointers: copied by the library on its stream).
"""
from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from . import _lib
from ._lib import (WLR_F32, WLR_F64, WLR_INIT_GHS, WLR_INIT_GIVEN, WlrError, check, lib,  # noqa: F401
                   wlr_opts)

__all__ = ["wlr_init", "wlr_iterate", "wlr_iterate_async", "wlr_sync", "wlr_objective",
           "wlr_trace", "wlr_result", "wlr_debug_state", "wlr_profile", "wlr_nccl_unique_id",
           "wlr_destroy", "wlr_version", "wlr_vgroup_create", "Handle", "VGroup", "WlrError", "LIB_PATH"]

LIB_PATH = _lib.LIB_PATH


def _ptr(x):
    """(pointer, dtype_code, is_device, keepalive) of a numpy array or torch tensor."""
    if x is None:
        return None, None, False, None
    try:
        import torch
        if isinstance(x, torch.Tensor):
            if not x.is_contiguous():
                x = x.contiguous()
            if x.dtype == torch.float32:
                code = WLR_F32
            elif x.dtype == torch.float64:
                code = WLR_F64
            else:
                raise TypeError(f"unsupported dtype {x.dtype}")
            return x.data_ptr(), code, x.is_cuda, x
    except ImportError:  # pragma: no cover
        pass
    a = np.ascontiguousarray(x)
    if a.dtype == np.float32:
        code = WLR_F32
    elif a.dtype == np.float64:
        code = WLR_F64
    else:
        raise TypeError(f"unsupported dtype {a.dtype}")
    return a.ctypes.data, code, False, a


class Handle:
    """Opaque wlr_handle plus the Python objects it borrows."""

    def __init__(self, raw, dims, dtype, keep):
        self.raw = raw
        self.m, self.n, self.k, self.r = dims
        self.dtype = dtype
        self._keep = keep

    @property
    def np_dtype(self):
        return np.float64 if self.dtype == WLR_F64 else np.float32

    def __del__(self):
        try:
            if getattr(self, "raw", None) and lib is not None:
                lib.wlr_destroy(self.raw)
                self.raw = None
        except Exception:  # interpreter shutdown
            pass


def wlr_init(A, k: int, r: int, W1=None, *, w1: float = 1.0, init: str = "ghs", x1_0=None,
             eps: float = 0.0, eig_tol: float = 0.0, eig_block: int = 0, eig_max_outer: int = 0,
             m_global: int = 0, row_offset: int = 0, nranks: int = 1, rank: int = 0,
             nccl_id: Optional[bytes] = None, stream: Optional[int] = None, use_graph: bool = True,
             seed: int = 0, vgroup: Optional["VGroup"] = None, check_every: int = 0) -> Handle:
    """wlr_init: PAPER.md Algorithm 1 lines 1-2 plus the first (C, D) half-step.
    ``W1=None`` uses the uniform weight ``w1``.  ``stream`` is a raw cudaStream_t (e.g.
    ``torch.cuda.current_stream().cuda_stream``); None lets the handle own a stream."""
    pa, code, _, ka = _ptr(A)
    m, n = (A.shape[0], A.shape[1])
    pw, wcode, _, kw = _ptr(W1)
    if W1 is not None and wcode != code:
        raise TypeError("A and W1 must have the same dtype")
    o = wlr_opts()
    lib.wlr_opts_default(ctypes.byref(o))
    o.dtype = code
    o.w1_scalar = float(w1)
    o.eps = float(eps)
    o.eig_tol = float(eig_tol)
    o.eig_block = int(eig_block)
    o.eig_max_outer = int(eig_max_outer)
    o.m_global = int(m_global)
    o.row_offset = int(row_offset)
    o.nranks = int(nranks)
    o.rank = int(rank)
    o.use_graph = 1 if use_graph else 0
    o.seed = int(seed)
    o.check_every = int(check_every)
    kx = None
    if init == "given":
        px, xcode, _, kx = _ptr(x1_0)
        if xcode != code:
            raise TypeError("x1_0 must have A's dtype")
        o.init = WLR_INIT_GIVEN
        o.x1_0 = px
    elif init != "ghs":
        raise ValueError("init must be 'ghs' or 'given'")
    idbuf = None
    if nccl_id is not None:
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        o.nccl_id = ctypes.cast(idbuf, ctypes.c_void_p)
    if stream is not None:
        o.stream = int(stream)
    if vgroup is not None:
        o.vgroup = vgroup.raw
    raw = ctypes.c_void_p()
    st = lib.wlr_init(ctypes.byref(raw), pa, A.shape[1] if A.ndim == 2 else n, pw,
                      (W1.shape[1] if W1 is not None else 0), m, n, int(k), int(r), ctypes.byref(o))
    check(st)
    return Handle(raw, (m, n, int(k), int(r)), code, (ka, kw, kx, idbuf))


class VGroup:
    """wlr_vgroup: G virtual ranks on one GPU (include/wlr.h); members are handles created with
    ``vgroup=``, ``nranks=G``, ``rank=g`` and driven from G host threads."""

    def __init__(self, G: int):
        self.raw = ctypes.c_void_p()
        self.G = int(G)
        check(lib.wlr_vgroup_create(self.G, ctypes.byref(self.raw)))

    def __del__(self):
        try:
            if getattr(self, "raw", None) and lib is not None:
                lib.wlr_vgroup_destroy(self.raw)
                self.raw = None
        except Exception:  # interpreter shutdown
            pass


def wlr_vgroup_create(G: int) -> VGroup:
    return VGroup(G)


def wlr_iterate(h: Handle, max_iters: int):
    """wlr_iterate: up to ``max_iters`` sWLR iterations; returns (iters_done, converged)."""
    done = ctypes.c_int32()
    conv = ctypes.c_int32()
    check(lib.wlr_iterate(h.raw, int(max_iters), ctypes.byref(done), ctypes.byref(conv)), h.raw)
    return done.value, bool(conv.value)


def wlr_iterate_async(h: Handle, n_iters: int):
    check(lib.wlr_iterate_async(h.raw, int(n_iters)), h.raw)


def wlr_sync(h: Handle):
    check(lib.wlr_sync(h.raw), h.raw)


def wlr_objective(h: Handle):
    """(F_p, ||X_p - X_{p-1}||_F, relative error) of the current canonical state."""
    f, s, r = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    check(lib.wlr_objective(h.raw, ctypes.byref(f), ctypes.byref(s), ctypes.byref(r)), h.raw)
    return f.value, s.value, r.value


def wlr_trace(h: Handle, cap: int = 4096) -> np.ndarray:
    """Trace rows (F_p, step, rel, p) for the last min(cap, states) canonical states."""
    out = np.zeros((cap, 4), dtype=np.float64)
    cnt = ctypes.c_int32()
    check(lib.wlr_trace(h.raw, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), cap,
                        ctypes.byref(cnt)), h.raw)
    return out[: cnt.value].copy()


def _host_out(shape, dtype):
    """Output array in page-locked host memory (device->host copies into pageable numpy memory run
    at ~2 GB/s); plain numpy when torch / CUDA is unavailable."""
    try:
        import torch
        if torch.cuda.is_available():
            tdt = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}[np.dtype(dtype)]
            return torch.empty(tuple(shape), dtype=tdt, pin_memory=True).numpy()
    except Exception:
        pass
    return np.empty(shape, dtype=dtype)


def wlr_result(h: Handle, x2: bool = False, b: bool = True):
    """Host copies of X1 (m x k), C (k x (n-k)), B (m x (r-k)), D = V^T ((r-k) x (n-k))
    and optionally X2 = X1 C + B D."""
    m, n, k, r = h.m, h.n, h.k, h.r
    dt = h.np_dtype
    X1 = _host_out((m, k), dt)
    C = _host_out((k, n - k), np.float64)
    B = _host_out((m, r - k), dt) if b else None
    D = _host_out((r - k, n - k), np.float64)
    X2 = _host_out((m, n - k), dt) if x2 else None
    check(lib.wlr_result(h.raw, X1.ctypes.data, k, C.ctypes.data, None if B is None else B.ctypes.data,
                         r - k, D.ctypes.data, None if X2 is None else X2.ctypes.data, n - k), h.raw)
    return dict(X1=X1, C=C, B=B, D=D, X2=X2)


def wlr_als_iterate(h: Handle, n_iters: int) -> np.ndarray:
    """f3 block ALS (R21) from the GHS state: runs n_iters sweeps and
    returns the objectives F_0 .. F_N of all states so far."""
    cap = 1 << 16
    F = np.zeros(cap, dtype=np.float64)
    check(lib.wlr_als_iterate(h.raw, int(n_iters), F.ctypes.data, cap), h.raw)
    h._als_states = getattr(h, "_als_states", 1) + int(n_iters)
    return F[: h._als_states].copy()


def wlr_als_iterate_async(h: Handle, n_iters: int) -> None:
    """Enqueue n_iters block-ALS sweeps without synchronising (F trace not copied)."""
    check(lib.wlr_als_iterate(h.raw, int(n_iters), None, 0), h.raw)
    h._als_states = getattr(h, "_als_states", 1) + int(n_iters)


def wlr_als_result(h: Handle):
    """Host copies of the block-ALS state: X1 (m x k), C (k x (n-k)), B (m x (r-k)), D ((r-k) x (n-k))."""
    m, n, k, r = h.m, h.n, h.k, h.r
    dt = h.np_dtype
    X1 = _host_out((m, k), dt)
    C = _host_out((k, n - k), np.float64)
    B = _host_out((m, r - k), dt)
    D = _host_out((r - k, n - k), np.float64)
    check(lib.wlr_als_result(h.raw, X1.ctypes.data, k, C.ctypes.data, B.ctypes.data, r - k, D.ctypes.data), h.raw)
    return dict(X1=X1, C=C, B=B, D=D)


def wlr_row_path(h: Handle, tensor_cores: bool) -> bool:
    """Select the row-pass implementation for uniform-weight fp32 problems: the tcgen05 3xTF32
    kernel (default) or the CUDA-core FP32 kernel.  Returns whether the tensor-core path is
    active afterwards (it is only available for uniform W1 with fp32 data)."""
    cnt = ctypes.c_int64()
    name = b"rowtc_on" if tensor_cores else b"rowtc_off"
    check(lib.wlr_debug_state(h.raw, name, None, 0, ctypes.byref(cnt)), h.raw)
    return bool(cnt.value)


def wlr_incr_path(h: Handle, tensor_cores: bool) -> bool:
    """Select the Gram-increment implementation for fp32 problems with k <= 32: the tcgen05
    3xTF32 kernel (default; used on the device only while the X1 step is small, R20)
    or always the CUDA-core FP32 kernel.  Returns whether the tensor-core kernel is enabled."""
    cnt = ctypes.c_int64()
    name = b"incrtc_on" if tensor_cores else b"incrtc_off"
    check(lib.wlr_debug_state(h.raw, name, None, 0, ctypes.byref(cnt)), h.raw)
    return bool(cnt.value)


def wlr_debug_state(h: Handle, name: str) -> np.ndarray:
    cnt = ctypes.c_int64()
    check(lib.wlr_debug_state(h.raw, name.encode(), None, 0, ctypes.byref(cnt)), h.raw)
    out = np.zeros(max(cnt.value, 8), dtype=np.float64)
    check(lib.wlr_debug_state(h.raw, name.encode(), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                              out.size, ctypes.byref(cnt)), h.raw)
    return out[: cnt.value] if name != "scal" else out


def wlr_profile(h: Handle, enable: bool, reset: bool = False):
    """Per-kernel device time (ms, CUDA events on the handle's streams) accumulated while
    profiling was enabled: row pass, increment GEMM, reduce, small step (critical half K3a)
    and the deferred small-step half (K3b, overlapped with the next row pass)."""
    ms = (ctypes.c_double * 6)()
    la = ctypes.c_int64()
    it = ctypes.c_int64()
    check(lib.wlr_profile(h.raw, 1 if enable else 0, 1 if reset else 0, ms, 6, ctypes.byref(la),
                          ctypes.byref(it)), h.raw)
    return dict(row_pass=ms[0], increments=ms[1], reduce=ms[2], small_step=ms[3], deferred=ms[4],
                row_solve=ms[5], launches=la.value, iters=it.value)


def wlr_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(lib.wlr_nccl_unique_id(buf))
    return buf.raw


def wlr_destroy(h: Handle):
    if h.raw:
        lib.wlr_destroy(h.raw)
        h.raw = None


def wlr_version() -> int:
    return lib.wlr_version()
