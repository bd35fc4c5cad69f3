"""The row-sharded path on ONE GPU through virtual ranks
(include/wlr.h wlr_vgroup): G handles over contiguous row shards (synth.shard_rows), each driven by
its own host thread like one process per GPU, the cross-rank sums done by the library's
fixed-order device reduce in place of NCCL.  Checked: X (all shards reassembled) and every F_p
against the fp64 oracle at the north-star tolerances, and the replicated state -- C, V, the whole
objective trace -- BITWISE identical on every member (PAPER.md:192 / Algorithm 1 line 7: rows are
independent given (C_p, D_p), so only the Gram sums are exchanged)."""
import dataclasses
import threading

import numpy as np
import pytest

import synth
from tests import gpu_util as gu

pytestmark = pytest.mark.gpu


def _run_group(cfg, A, W1, G, iters):
    import torch
    w = gu.need_gpu()
    grp = w.wlr_vgroup_create(G)
    out = [None] * G
    errs = []

    def member(g):
        try:
            torch.cuda.set_device(0)
            r0, r1 = synth.shard_rows(cfg.m, G, g)
            At = torch.from_numpy(np.ascontiguousarray(A[r0:r1])).cuda()
            Wt = None if W1 is None else torch.from_numpy(np.ascontiguousarray(W1[r0:r1])).cuda()
            h = w.wlr_init(At, cfg.k, cfg.r, Wt, w1=cfg.w_const or 1.0, m_global=cfg.m, row_offset=r0,
                           nranks=G, rank=g, vgroup=grp)
            w.wlr_iterate(h, iters)
            res = w.wlr_result(h, x2=True)
            res["trace"] = w.wlr_trace(h)
            res["V"] = w.wlr_debug_state(h, "V")
            res["keep"] = (At, Wt, h)
            out[g] = res
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)

    th = [threading.Thread(target=member, args=(g,)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    assert all(o is not None for o in out)
    return out


def _check(cfg, A, W1, G, iters):
    out = _run_group(cfg, A, W1, G, iters)
    for g in range(1, G):                                       # replicated state: bitwise
        np.testing.assert_array_equal(out[g]["C"], out[0]["C"])
        np.testing.assert_array_equal(out[g]["V"], out[0]["V"])
        np.testing.assert_array_equal(out[g]["trace"], out[0]["trace"])
    X = np.concatenate([np.concatenate([o["X1"], o["X2"]], axis=1) for o in out], axis=0).astype(np.float64)
    o = gu.run_oracle(cfg, A, W1, iters)
    ex = gu.rel(X, o.x)
    assert ex <= gu.TOL_X[cfg.dtype], ex
    fo = np.array([rec["F"] for rec in o.trace])
    ef = np.abs(out[0]["trace"][:, 0] - fo) / np.abs(fo)
    assert ef.max() <= gu.TOL_F[cfg.dtype], ef.max()
    return ex, float(ef.max())


@pytest.mark.parametrize("G", [2, 3, 8])
def test_virtual_shards_config1_fp64(G):
    """config 1 (fp64, uniform W1 = 50, incremental Grams): 300 rows over G ranks, 300/8 uneven."""
    cfg = synth.CONFIGS[1]
    A, W1 = gu.inputs(cfg)
    ex, ef = _check(cfg, A, W1, G, 12)
    print(f"G={G} config 1: relX {ex:.2e} relF {ef:.2e}")


@pytest.mark.parametrize("G", [2, 3, 8])
def test_virtual_shards_nonuniform_fp32(G):
    """scaled config 4 (fp32, log-uniform W1, per-row solves, per-iteration increment sums)."""
    cfg = dataclasses.replace(synth.scaled(synth.CONFIGS[4], 36, 48), iters=6)
    A, W1 = gu.inputs(cfg)
    ex, ef = _check(cfg, A, W1, G, cfg.iters)
    print(f"G={G} scaled config 4: relX {ex:.2e} relF {ef:.2e}")


@pytest.mark.parametrize("G", [2, 8])
def test_virtual_shards_uniform_fp32_propagation(G):
    """scaled config 3 (fp32, uniform W1: Gram propagation, nothing exchanged per iteration)."""
    cfg = dataclasses.replace(synth.scaled(synth.CONFIGS[3], 60, 80), n=120, iters=8)
    A, W1 = gu.inputs(cfg)
    ex, ef = _check(cfg, A, W1, G, cfg.iters)
    print(f"G={G} scaled config 3: relX {ex:.2e} relF {ef:.2e}")
