"""C-ABI checks that need no GPU (``-m "not gpu"``): libwlr.so loads, exports every entry
point include/wlr.h declares, and its host-side argument validation returns the documented
status codes before any device work (include/wlr.h "Errors"; PAPER.md:94 for r > k and
W1 > 0)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "wlr.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(wlr_[a-z_0-9]+)\s*\(", src)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_1703_06303_b200 import _lib
    return _lib


def test_header_declares_the_north_star_entry_points():
    names = declared_symbols()
    for must in ("wlr_init", "wlr_iterate", "wlr_objective", "wlr_result", "wlr_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    raw = ctypes.CDLL(lib.LIB_PATH)
    missing = [n for n in declared_symbols() if not hasattr(raw, n)]
    assert not missing, missing
    assert set(declared_symbols()) == set(lib.EXPORTS)


def test_version_and_status_strings(lib):
    assert lib.lib.wlr_version() >= 1
    for code, name in enumerate(["WLR_OK", "WLR_EINVAL", "WLR_ERANK", "WLR_EEIG", "WLR_EINTERNAL",
                                 "WLR_ENONFINITE", "WLR_ECUDA", "WLR_ENCCL", "WLR_ENOMEM"]):
        assert lib.lib.wlr_status_string(code).decode() == name


def test_opts_default(lib):
    o = lib.wlr_opts()
    lib.lib.wlr_opts_default(ctypes.byref(o))
    assert o.dtype == lib.WLR_F32 and o.init == lib.WLR_INIT_GHS and o.nranks == 1 and o.use_graph == 1
    assert o.w1_scalar == 1.0 and o.eps == 0.0


@pytest.mark.parametrize("m,n,k,r,msg", [
    (100, 20, 5, 5, "r > k"),          # Theorem 2 needs r > k
    (100, 20, 0, 3, "1 <= k < n"),
    (100, 20, 20, 22, "1 <= k < n"),
    (100, 20, 5, 21, "r <= min"),
])
def test_invalid_dimensions_fail_before_device_work(lib, m, n, k, r, msg):
    A = np.zeros((m, n), dtype=np.float32)
    h = ctypes.c_void_p()
    o = lib.wlr_opts()
    lib.lib.wlr_opts_default(ctypes.byref(o))
    st = lib.lib.wlr_init(ctypes.byref(h), A.ctypes.data, n, None, 0, m, n, k, r, ctypes.byref(o))
    assert st == lib.WLR_EINVAL
    assert msg in lib.lib.wlr_last_error(None).decode()
    assert not h.value


def test_uniform_weight_must_be_positive(lib):
    A = np.zeros((50, 10), dtype=np.float32)
    h = ctypes.c_void_p()
    o = lib.wlr_opts()
    lib.lib.wlr_opts_default(ctypes.byref(o))
    o.w1_scalar = 0.0                                   # W1 > 0
    st = lib.lib.wlr_init(ctypes.byref(h), A.ctypes.data, 10, None, 0, 50, 10, 3, 5, ctypes.byref(o))
    assert st == lib.WLR_EINVAL


def test_binding_refuses_to_run_without_the_library(tmp_path, monkeypatch):
    """No CPU fallback: the loader raises when libwlr.so is absent."""
    from paper_1703_06303_b200 import _lib
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        _lib._load()
