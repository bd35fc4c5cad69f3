"""Helpers for the ``-m gpu`` parity tests: run the CUDA path through the C ABI binding and
the fp64 oracle on the same seeded inputs, and compare (tolerances from BASELINE.json
north_star: relative Frobenius error of X <= 1e-4 (fp32) / 1e-10 (fp64), relative
objective error <= 1e-5)."""
import numpy as np
import pytest

import oracle
import synth
from oracle.swlr import assemble

TOL_X = {"f32": 1e-4, "f64": 1e-10}
TOL_F = {"f32": 1e-5, "f64": 1e-10}


def need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1703_06303_b200 as w  # noqa: F401  (fails loudly if libwlr.so is missing)
    return w


def inputs(cfg):
    A = synth.make_A(cfg)
    W1 = synth.make_W1(cfg)
    return A, W1


def run_gpu(cfg, A, W1, iters, device=True, tensor_cores=True, **kw):
    import torch
    w = need_gpu()
    if device:
        At = torch.from_numpy(A).cuda()
        Wt = None if W1 is None else torch.from_numpy(W1).cuda()
    else:
        At, Wt = A, W1
    h = w.wlr_init(At, cfg.k, cfg.r, Wt, w1=cfg.w_const or 1.0, **kw)
    tc = w.wlr_row_path(h, tensor_cores)
    tr0 = w.wlr_trace(h)
    if iters:
        done, conv = w.wlr_iterate(h, iters)
    res = w.wlr_result(h, x2=True)
    res["trace"] = w.wlr_trace(h)
    res["trace0"] = tr0
    res["handle"] = h
    res["keep"] = (At, Wt)
    res["tensor_cores"] = tc
    return res


def gpu_X(res):
    return np.concatenate([res["X1"].astype(np.float64), res["X2"].astype(np.float64)], axis=1)


def run_oracle(cfg, A, W1, iters, x1_0=None):
    w1 = synth.dense_W1(cfg, W1, cfg.m)
    return oracle.swlr(A.astype(np.float64), w1, cfg.k, cfg.r, iters=iters, x1_0=x1_0)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def compare(cfg, g, o, tol_x=None, tol_f=None, check_steps=True):
    tol_x = TOL_X[cfg.dtype] if tol_x is None else tol_x
    tol_f = TOL_F[cfg.dtype] if tol_f is None else tol_f
    X = gpu_X(g)
    ex = rel(X, o.x)
    assert ex <= tol_x, f"relX {ex:.3e} > {tol_x:.1e}"
    # the whole objective trace, state by state (R11: F_p of the canonical state)
    tr = g["trace"]
    fo = np.array([rec["F"] for rec in o.trace])
    assert tr.shape[0] == len(o.trace), (tr.shape, len(o.trace))
    ef = np.abs(tr[:, 0] - fo) / np.abs(fo)
    assert ef.max() <= tol_f, f"relF {ef.max():.3e} at p={int(ef.argmax())}"
    if check_steps:
        so = np.array([rec.get("step", -1.0) for rec in o.trace])
        ro = np.array([rec.get("rel", -1.0) for rec in o.trace])
        big = ro > (1e-5 if cfg.dtype == "f32" else 1e-10)
        big[0] = False
        if big.any():
            es = np.abs(tr[big, 1] - so[big]) / so[big]
            assert es.max() <= (2e-2 if cfg.dtype == "f32" else 1e-3), f"step mismatch {es.max():.3e}"
            # rel_p = Error_p / ||X_p|| (reading R3), element-wise
            er = np.abs(tr[big, 2] - ro[big]) / ro[big]
            assert er.max() <= (2e-2 if cfg.dtype == "f32" else 1e-3), f"rel mismatch {er.max():.3e}"
    return ex, float(ef.max())
