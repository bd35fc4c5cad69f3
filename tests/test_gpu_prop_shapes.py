"""GPU parity of the Gram-propagation path (uniform W1, fp32: prop1 / prop2) at
shapes that exercise its variants: rows per prop1 CTA RB = ceil(n / min(n, #SMs less the K3b / shadow clusters)) from 1 to 8
(uneven row splits), Q column blocks rounded to 2 / 8 / 16 (k = 8, 20..30, 36), r - k = 1..5, and
G_A Y computed in prop1 or left to the small step (Y not fitting in prop1's shared memory).
Against the fp64 oracle (literal Algorithm 1) on the same seeded inputs and iteration count."""
import dataclasses

import numpy as np
import pytest

import synth
from tests import gpu_util as gu

pytestmark = pytest.mark.gpu


def _lowrank(m, n, q, seed):
    """A = U diag(sigma) V + noise with decaying sigma (separated top singular values)."""
    g = np.random.default_rng(seed)
    U = np.linalg.qr(g.standard_normal((m, q)))[0]
    V = np.linalg.qr(g.standard_normal((n, q)))[0].T
    sig = 10.0 / (1.0 + np.arange(q)) ** 1.5
    return (U * sig) @ V + 1e-3 * g.standard_normal((m, n))


@pytest.mark.parametrize("m,n,k,r", [
    (2000, 100, 8, 9),       # RB 1, Q column blocks 2 -> 2, r - k = 1
    (1500, 200, 20, 22),     # RB 2 (uneven: 52 CTAs with 2 rows), ncb 5 -> 8
    (1200, 450, 36, 41),     # RB 4, ncb 9 -> 16 (RP 64), b = 7
    (1000, 700, 30, 31),     # RB 5 (config 3's), r - k = 1
    (800, 1030, 8, 12),      # RB 7; Y (n-k x 6) does not fit beside W' and the rows: G_A Y in the small step
])
def test_gram_propagation_shapes(m, n, k, r):
    import torch
    w = gu.need_gpu()
    A = _lowrank(m, n, r + 6, seed=1000 + n).astype(np.float32)
    cfg = dataclasses.replace(synth.CONFIGS[2], name="prop", m=m, n=n, k=k, r=r, w_const=30.0, iters=15)
    g = gu.run_gpu(cfg, A, None, cfg.iters)
    info = w.wlr_debug_state(g["handle"], "prop")
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    assert info[0] == 1.0, "Gram propagation not active"
    nsp = int(info[4])                        # SMs left to prop1 beside the K3b / shadow clusters
    assert 1 <= nsp <= nsm and info[5] == 1.0
    assert info[1] == min(n, nsp) and info[2] == -(-n // min(n, nsp))
    if n == 1030 and nsm == 148:
        assert info[3] == 0.0                  # (the G_A Y fallback inside the small step)
    o = gu.run_oracle(cfg, A, None, cfg.iters)
    gu.compare(cfg, g, o)


def test_n_minus_k_beyond_the_cluster_is_rejected():
    """n - k > 16 x 64 columns: an explicit WLR_EINVAL at init, not a launch failure."""
    import torch
    w = gu.need_gpu()
    A = torch.from_numpy(_lowrank(300, 1100, 20, seed=7).astype(np.float32)).cuda()
    with pytest.raises(w.WlrError) as e:
        w.wlr_init(A, 16, 18, None, w1=30.0)
    assert "n - k > 1024" in str(e.value)


@pytest.mark.parametrize("cfg_id", [2, 3])
def test_shadow_small_step_is_bitwise_neutral(cfg_id, monkeypatch):
    """The shadow K3a (a rerun of K3a(p-1) into private buffers at the start of iteration p, which
    warms K3a's code in L2) changes nothing: trace and result bitwise identical with
    it off, at the same prop1 grid (WLR_PROP_RSV fixed), over iterations that cross the graph phases
    and a host synchronisation (the eager p = 0 iteration and the shadow's own state chain)."""
    w = gu.need_gpu()
    import torch
    cfg = synth.CONFIGS[cfg_id]
    A = torch.from_numpy(synth.make_A(cfg)).cuda()
    out = {}
    for sh in ("0", "1"):
        monkeypatch.setenv("WLR_SHADOW", sh)
        monkeypatch.setenv("WLR_PROP_RSV", "32")
        h = w.wlr_init(A, cfg.k, cfg.r, None, w1=cfg.w_const)
        assert w.wlr_debug_state(h, "prop")[5] == float(sh)
        w.wlr_iterate(h, 7)
        w.wlr_iterate(h, 13)
        r = w.wlr_result(h, x2=False)
        out[sh] = (np.asarray(w.wlr_trace(h)).copy(), {k_: np.asarray(v).copy() for k_, v in r.items() if v is not None})
    assert np.array_equal(out["0"][0], out["1"][0])
    for k_ in out["0"][1]:
        assert np.array_equal(out["0"][1][k_], out["1"][1][k_]), k_
