"""The NCCL path on one B200: a one-rank communicator (wlr_nccl_unique_id + nranks = 1) routes the
init Gram sums and, for non-uniform W1, the per-iteration increment sum [N, Gamma, Omega, f_w]
(captured into the iteration's CUDA graph) through ncclAllReduce.  A one-rank sum is the identity,
so the run must be BITWISE identical to the same run without a communicator (the
multi-GPU data path is the sharded row pass + this allreduce)."""
import dataclasses

import numpy as np
import pytest

import synth
from tests import gpu_util as gu

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ci", [2, 4])
def test_one_rank_nccl_communicator_is_bitwise_neutral(ci):
    import torch
    w = gu.need_gpu()
    cfg = synth.CONFIGS[ci] if ci == 2 else dataclasses.replace(synth.scaled(synth.CONFIGS[4], 60, 80), iters=8)
    A, W1 = gu.inputs(cfg)
    At = torch.from_numpy(A).cuda()
    Wt = None if W1 is None else torch.from_numpy(W1).cuda()
    out = []
    for nccl in (False, True):
        kw = dict(nranks=1, rank=0, nccl_id=w.wlr_nccl_unique_id()) if nccl else {}
        h = w.wlr_init(At, cfg.k, cfg.r, Wt, w1=cfg.w_const or 1.0, **kw)
        w.wlr_iterate(h, 8)
        res = w.wlr_result(h, x2=True)
        out.append((w.wlr_trace(h), res["X1"], res["C"]))
        w.wlr_destroy(h)
    for a, b in zip(out[0], out[1]):
        np.testing.assert_array_equal(a, b)
