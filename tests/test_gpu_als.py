"""GPU parity of the f3 block ALS (R21) through the C ABI
(wlr_als_iterate / wlr_als_result) against the fp64 oracle oracle/block_als.py on the same seeded
inputs: objective of every state and the final X = (X1, X1 C + B D)."""
import dataclasses

import numpy as np
import pytest

import synth
from oracle import block_als
from tests import gpu_util as gu

pytestmark = pytest.mark.gpu


def _run(cfg, A, W1, iters):
    import torch
    w = gu.need_gpu()
    At = torch.from_numpy(A).cuda()
    Wt = None if W1 is None else torch.from_numpy(W1).cuda()
    h = w.wlr_init(At, cfg.k, cfg.r, Wt, w1=cfg.w_const or 1.0)
    F = w.wlr_als_iterate(h, iters)
    res = w.wlr_als_result(h)
    res["F"] = F
    res["handle"] = h
    res["keep"] = (At, Wt)
    return res


def _compare(cfg, A, W1, iters):
    g = _run(cfg, A, W1, iters)
    w1 = synth.dense_W1(cfg, W1, cfg.m)
    o = block_als.block_als(A.astype(np.float64), w1, cfg.k, cfg.r, iters)
    fo = np.array([rec["F"] for rec in o.trace])
    assert g["F"].shape == fo.shape
    ef = np.abs(g["F"] - fo) / np.abs(fo)
    assert ef.max() <= gu.TOL_F[cfg.dtype], (ef.max(), ef.argmax())
    X1 = g["X1"].astype(np.float64)
    Xg = np.concatenate([X1, X1 @ g["C"] + g["B"].astype(np.float64) @ g["D"]], axis=1)
    Xo = np.concatenate([o.x1, o.x1 @ o.c + o.b @ o.d], axis=1)
    ex = gu.rel(Xg, Xo)
    assert ex <= gu.TOL_X[cfg.dtype], ex
    # the ALS objective never increases (exact block minimisations), on the GPU too
    assert np.all(np.diff(g["F"]) <= 1e-9 * g["F"][0]) if cfg.dtype == "f64" else True
    return g, o


def test_als_config1_fp64():
    cfg = synth.CONFIGS[1]
    A, W1 = gu.inputs(cfg)
    _compare(cfg, A, W1, 20)


def test_als_config2_fp32():
    cfg = synth.CONFIGS[2]
    A, W1 = gu.inputs(cfg)
    _compare(cfg, A, W1, 15)


def test_als_nonuniform_fp64_tiny():
    g0 = np.random.default_rng(11)
    cfg = dataclasses.replace(synth.CONFIGS[1], w_const=None)
    A = synth.make_A(cfg)
    W1 = np.exp(g0.uniform(np.log(2.0), np.log(300.0), (cfg.m, cfg.k)))
    _compare(cfg, A, W1, 12)


def test_als_nonuniform_fp32_scaled_config4():
    cfg = dataclasses.replace(synth.scaled(synth.CONFIGS[4], 48, 64), iters=6)
    A, W1 = gu.inputs(cfg)
    _compare(cfg, A, W1, 6)


def test_als_consumes_the_swlr_state():
    w = gu.need_gpu()
    cfg = synth.CONFIGS[1]
    A, W1 = gu.inputs(cfg)
    g = _run(cfg, A, W1, 2)
    with pytest.raises(w.WlrError) as e:
        w.wlr_iterate(g["handle"], 1)
    assert e.value.status == 1


def test_als_rejects_r_minus_k_wider_than_x1_rows():
    """B shares X1's kp-wide row layout: r - k > round_up(k, 4) is rejected with WLR_EINVAL
    instead of writing past the B buffer."""
    import torch
    w = gu.need_gpu()
    g = np.random.default_rng(5)
    A = g.standard_normal((200, 30))
    h = w.wlr_init(torch.from_numpy(A).cuda(), 4, 12, None, w1=10.0)   # r - k = 8 > kp = 4
    with pytest.raises(w.WlrError) as ei:
        w.wlr_als_iterate(h, 1)
    assert "r - k" in str(ei.value)
