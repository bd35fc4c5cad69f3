"""Pins of the f3 oracle (oracle/block_als.py, R21): properties the paper and the
mathematics fix -- monotone objective under exact block minimisation, stationarity (normal
equations) of every block step, Theorem 1 at p = 0, and the order relation with sWLR's exact
(C, D) step (Theorem 2)."""
import numpy as np
import pytest

import oracle
from oracle import block_als as ba


def _problem(seed, m=60, n=14, k=4, r=7, wlo=2.0, whi=40.0, lowrank=None):
    g = np.random.default_rng(seed)
    if lowrank:
        a = g.standard_normal((m, lowrank)) @ g.standard_normal((lowrank, n))
    else:
        a = g.standard_normal((m, 3)) @ g.standard_normal((3, n)) + 0.3 * g.standard_normal((m, n))
    w1 = np.exp(g.uniform(np.log(wlo), np.log(whi), (m, k)))
    return a, w1, k, r


def test_ghs_start_is_theorem1():
    """p = 0: X1_0 C_0 + B_0 D_0 = A~2 of Theorem 1, and rank(B_0 D_0) = r - k."""
    a, w1, k, r = _problem(0)
    a1, a2 = a[:, :k], a[:, k:]
    c, b, d = ba.ghs_factors(a1, a2, r)
    np.testing.assert_allclose(a1 @ c + b @ d, oracle.ghs_solve(a1, a2, r), atol=1e-11)
    assert np.linalg.matrix_rank(b @ d, tol=1e-9) == r - k


def test_objective_is_monotone_through_every_block_step():
    """Each block update is the exact minimiser of a convex quadratic in that block, so F never
    increases along the sweep (sub-step by sub-step)."""
    a, w1, k, r = _problem(1)
    res = ba.block_als(a, w1, k, r, iters=25)
    f = [res.trace[0]["F"]]
    for rec in res.trace[1:]:
        f += [rec["F_x1"], rec["F_c"], rec["F_b"], rec["F"]]
    f = np.array(f)
    assert np.all(np.diff(f) <= 1e-12 * f[0]), np.diff(f).max()
    assert f[-1] < f[0]


def test_each_block_step_is_stationary():
    """Normal equations of each least-squares step, and the X1 gradient of PAPER.md:190."""
    a, w1, k, r = _problem(2)
    a1, a2 = a[:, :k], a[:, k:]
    c, b, d = ba.ghs_factors(a1, a2, r)
    x1 = oracle.x1_step(a1, a2, w1, c, b @ d)
    # -(A1 - X1) . W1 . W1 - (A2 - X1 C_p - D_p) C_p^T = 0 with D_p = B_p D_p
    grad = -(a1 - x1) * w1 * w1 - (a2 - x1 @ c - b @ d) @ c.T
    assert np.abs(grad).max() <= 1e-9 * np.abs(a).max() ** 2
    c2 = ba.c_step(x1, a2, b, d)
    assert np.abs(x1.T @ (a2 - x1 @ c2 - b @ d)).max() <= 1e-9 * np.abs(a).max() ** 2
    b2 = ba.b_step(x1, c2, a2, d)
    assert np.abs((a2 - x1 @ c2 - b2 @ d) @ d.T).max() <= 1e-9 * np.abs(a).max() ** 2
    d2 = ba.d_step(x1, c2, a2, b2)
    assert np.abs(b2.T @ (a2 - x1 @ c2 - b2 @ d2)).max() <= 1e-9 * np.abs(a).max() ** 2


def test_swlr_exact_cd_step_is_never_worse_than_the_als_sweep():
    """For the same X1, sWLR's (C, D) (Theorem 2: the joint minimiser over C and rank-(r-k) D)
    gives an objective <= the one-sweep (C, B, D) update of R21 (a cross-pin between the oracles)."""
    a, w1, k, r = _problem(3)
    a1, a2 = a[:, :k], a[:, k:]
    res = ba.block_als(a, w1, k, r, iters=3)
    x1 = res.x1
    c_s, d_s, _ = oracle.cd_step(x1, a2, r)
    f_swlr = oracle.objective(a1, a2, w1, x1, c_s, d_s)
    f_als = res.trace[-1]["F"]
    assert f_swlr <= f_als * (1 + 1e-12)


def test_exactly_representable_data_stays_at_zero():
    """rank(A) <= r with full-rank A1: the GHS point already has F = 0 and every sweep keeps it."""
    a, w1, k, r = _problem(4, lowrank=6)
    res = ba.block_als(a, w1, k, r, iters=5)
    scale = float(np.sum(a * a))
    assert all(rec["F"] <= 1e-20 * scale for rec in res.trace)


def test_converged_point_is_stationary_in_all_blocks():
    """After many sweeps the iterate is a stationary point of F in all four blocks at once."""
    a, w1, k, r = _problem(5, m=40, n=10, k=3, r=5)
    a1, a2 = a[:, :k], a[:, k:]
    res = ba.block_als(a, w1, k, r, iters=3000)
    x1, c, b, d = res.x1, res.c, res.b, res.d
    resid = a2 - x1 @ c - b @ d
    sc = np.abs(a).max() ** 2
    assert np.abs(-(a1 - x1) * w1 * w1 - resid @ c.T).max() <= 1e-6 * sc      # d/dX1
    assert np.abs(x1.T @ resid).max() <= 1e-6 * sc                           # d/dC
    assert np.abs(resid @ d.T).max() <= 1e-6 * sc                            # d/dB
    assert np.abs(b.T @ resid).max() <= 1e-6 * sc                            # d/dD


def test_input_validation():
    a, w1, k, r = _problem(6)
    with pytest.raises(ValueError):
        ba.block_als(a, w1, k, k, iters=1)
    w0 = w1.copy()
    w0[0, 0] = 0.0
    with pytest.raises(ValueError):
        ba.block_als(a, w0, k, r, iters=1)
