"""Pins for ``oracle/swlr_large.py`` (the m >= 1e5 restatement of Algorithm 1 used for the
config-5 fixture; reading R22), CPU only.

* Against the literal oracle ``oracle.swlr`` (pinned itself by P1-P12) on inputs where both run:
  the same states X_p, F_p, Error_p and rel_p (configs 1, 2 and scaled 4 / 5, uniform and
  non-uniform W1, fp64 and fp32-rounded data).
* Directly against the paper: Theorem 1 at p = 0, monotone half-steps
  (each half-step is an exact minimisation), the Theorem-2 fixed point of every
  canonical state, and D = U (Sigma)_{r-k} V^T through an independent SVD.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle.swlr_large import cd_step_gram, swlr_large

import concurrent.futures as cf


def _cases():
    yield synth.CONFIGS[1]
    yield synth.scaled(synth.CONFIGS[2], 30, 40)
    yield synth.scaled(synth.CONFIGS[4], 24, 32)
    yield synth.scaled(synth.CONFIGS[5], 72, 128)


@pytest.mark.parametrize("cfg", list(_cases()), ids=lambda c: c.name)
def test_large_route_matches_literal_oracle(cfg):
    A = synth.make_A(cfg)
    W1 = synth.make_W1(cfg)
    w1 = synth.dense_W1(cfg, W1, cfg.m)
    iters = 4
    o = oracle.swlr(A.astype(np.float64), w1, cfg.k, cfg.r, iters=iters)
    g = swlr_large(A, W1, cfg.k, cfg.r, iters, w_const=cfg.w_const or 1.0, threads=2)
    X = g.x_rows(np.arange(cfg.m))
    assert np.linalg.norm(X - o.x) <= 1e-10 * np.linalg.norm(o.x)
    for a, b in zip(o.trace, g.trace):
        assert abs(a["F"] - b["F"]) <= 1e-11 * a["F"]
        if a["p"] > 0:
            assert abs(a["F_mid"] - b["F_mid"]) <= 1e-11 * a["F_mid"]
            if a["rel"] > 1e-8:          # below that the step is rounding noise in both routes
                assert abs(a["rel"] - b["rel"]) <= 1e-6 * a["rel"]
                assert abs(a["step"] - b["step"]) <= 1e-6 * a["step"]
        np.testing.assert_allclose(b["sig_t"], a["sig_t"], rtol=1e-10)


def test_large_route_theorem1_and_svd_form_of_D():
    """p = 0 is Theorem 1; the eigh(P^T P) triplets give D = U Sigma_{r-k} V^T of an SVD."""
    cfg = synth.scaled(synth.CONFIGS[5], 72, 128)
    A = synth.make_A(cfg).astype(np.float64)
    k, r = cfg.k, cfg.r
    a1, a2 = A[:, :k], A[:, k:]
    with cf.ThreadPoolExecutor(2) as pool:
        st = cd_step_gram(a1.copy(), A, k, r, pool)
    # Theorem 1 through an SVD basis of A1 (not the QR the oracle uses)
    u1, _, _ = np.linalg.svd(a1, full_matrices=False)
    pa2 = u1 @ (u1.T @ a2)
    u, s, vt = np.linalg.svd(a2 - pa2, full_matrices=False)
    t = r - k
    ghs = pa2 + (u[:, :t] * s[:t]) @ vt[:t]
    x2 = a1 @ st.c + st.b @ st.vt
    assert np.linalg.norm(x2 - ghs) <= 1e-10 * np.linalg.norm(ghs)
    np.testing.assert_allclose(st.sigma[: t + 1], s[: t + 1], rtol=1e-9)
    # V has orthonormal rows
    np.testing.assert_allclose(st.vt @ st.vt.T, np.eye(t), atol=1e-12)


def test_large_route_monotone_and_fixed_point():
    """Each half-step is an exact minimisation: F_mid <= F_p, F_{p+1} <= F_mid;
    and X2_p = P_{X1} A2 + H_{r-k}(P^perp A2) at every canonical state (Theorem 2)."""
    cfg = synth.scaled(synth.CONFIGS[4], 24, 32)
    A = synth.make_A(cfg)
    W1 = synth.make_W1(cfg)
    g = swlr_large(A, W1, cfg.k, cfg.r, 6, threads=2)
    F = [rec["F"] for rec in g.trace]
    for p in range(1, len(F)):
        fm = g.trace[p]["F_mid"]
        assert fm <= F[p - 1] * (1 + 1e-12) and F[p] <= fm * (1 + 1e-12)
    a = A.astype(np.float64)
    k = cfg.k
    x1 = g.x1
    q, _ = np.linalg.qr(x1)
    pa2 = q @ (q.T @ a[:, k:])
    ref = pa2 + oracle.hard_threshold(a[:, k:] - pa2, cfg.r - k)
    x2 = g.x_rows(np.arange(cfg.m))[:, k:]
    assert np.linalg.norm(x2 - ref) <= 1e-9 * (1 + np.linalg.norm(a[:, k:]))
