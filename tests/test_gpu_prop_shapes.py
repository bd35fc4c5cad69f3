"""GPU parity of the Gram-propagation path (uniform W1, fp32: prop1 / prop2) at
shapes that exercise its variants: rows per prop1 CTA RB = ceil(n / min(n, #SMs)) from 1 to 8
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
    assert info[1] == min(n, nsm) and info[2] == -(-n // min(n, nsm))
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
