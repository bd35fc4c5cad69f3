"""ctypes binding of libwlr.so (include/wlr.h).  Argument marshalling only: every step of
the sWLR iteration runs in the library's CUDA kernels.  Importing this module fails loudly
when the library has not been built -- there is no Python or CPU fallback."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libwlr.so")

WLR_OK, WLR_EINVAL, WLR_ERANK, WLR_EEIG, WLR_EINTERNAL, WLR_ENONFINITE, WLR_ECUDA, WLR_ENCCL, WLR_ENOMEM = range(9)
WLR_F32, WLR_F64 = 0, 1
WLR_INIT_GHS, WLR_INIT_GIVEN = 0, 1

# every symbol include/wlr.h declares
EXPORTS = ("wlr_opts_default", "wlr_init", "wlr_iterate", "wlr_iterate_async", "wlr_sync",
           "wlr_objective", "wlr_trace", "wlr_result", "wlr_debug_state", "wlr_profile",
           "wlr_nccl_unique_id", "wlr_last_error", "wlr_status_string", "wlr_destroy",
           "wlr_version", "wlr_als_iterate", "wlr_als_result", "wlr_vgroup_create", "wlr_vgroup_destroy")


class wlr_opts(ctypes.Structure):
    _fields_ = [
        ("dtype", ctypes.c_int32),
        ("init", ctypes.c_int32),
        ("x1_0", ctypes.c_void_p),
        ("w1_scalar", ctypes.c_double),
        ("eps", ctypes.c_double),
        ("eig_tol", ctypes.c_double),
        ("eig_block", ctypes.c_int32),
        ("eig_max_outer", ctypes.c_int32),
        ("m_global", ctypes.c_int64),
        ("row_offset", ctypes.c_int64),
        ("nranks", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("nccl_id", ctypes.c_void_p),
        ("stream", ctypes.c_void_p),
        ("use_graph", ctypes.c_int32),
        ("seed", ctypes.c_int32),
        ("vgroup", ctypes.c_void_p),
        ("check_every", ctypes.c_int32),
    ]


class WlrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{status_string(status)}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_1703_06303_b200/build.py` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    P = ctypes.POINTER
    sig = {
        "wlr_opts_default": (None, [P(wlr_opts)]),
        "wlr_init": (i32, [P(vp), vp, i64, vp, i64, i64, i64, i64, i64, P(wlr_opts)]),
        "wlr_iterate": (i32, [vp, i32, P(i32), P(i32)]),
        "wlr_iterate_async": (i32, [vp, i32]),
        "wlr_sync": (i32, [vp]),
        "wlr_objective": (i32, [vp, P(dbl), P(dbl), P(dbl)]),
        "wlr_trace": (i32, [vp, P(dbl), i32, P(i32)]),
        "wlr_result": (i32, [vp, vp, i64, vp, vp, i64, vp, vp, i64]),
        "wlr_debug_state": (i32, [vp, ctypes.c_char_p, P(dbl), i64, P(i64)]),
        "wlr_profile": (i32, [vp, i32, i32, P(dbl), i32, P(i64), P(i64)]),
        "wlr_nccl_unique_id": (i32, [vp]),
        "wlr_last_error": (ctypes.c_char_p, [vp]),
        "wlr_status_string": (ctypes.c_char_p, [i32]),
        "wlr_destroy": (None, [vp]),
        "wlr_version": (i32, []),
        "wlr_als_iterate": (i32, [vp, i32, vp, i32]),
        "wlr_als_result": (i32, [vp, vp, i64, vp, vp, i64, vp]),
        "wlr_vgroup_create": (i32, [i32, P(vp)]),
        "wlr_vgroup_destroy": (None, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def status_string(s: int) -> str:
    return lib.wlr_status_string(int(s)).decode()


def last_error(h=None) -> str:
    r = lib.wlr_last_error(h)
    return r.decode() if r else ""


def check(status: int, h=None):
    if status != WLR_OK:
        raise WlrError(status, last_error(h))
