"""Pins P1-P12 for the oracle's Algorithm 1 (CPU, ``-m "not gpu"``).

Each test fixes the oracle against something other than itself: a closed form
(Theorem 1, Eq. (2)), an invariant the paper states (monotone half-steps, rank
bound, Theorem 2 fixed point, stationarity Eq. after), a hand-worked
fixture, or brute force (general ALS).  A plausible mistake anywhere in
``oracle/swlr.py`` (a dropped term in E, a transposed C, a wrong row weight, a
stale C_p in the output, a wrong truncation rank) fails at least one of them.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle.swlr import assemble
from tests import gram_route
from tests.golden_io import load


def cfg1_data(w=50.0):
    cfg = synth.CONFIGS[1]
    a = synth.make_A(cfg).astype(np.float64)
    return cfg, a, np.full((cfg.m, cfg.k), w)


def ghs_by_svd(a1, a2, r):
    """Theorem 1 evaluated through an SVD-based basis of A1 (independent of the
    oracle's QR route) and numpy's SVD truncation."""
    u1, s1, _ = np.linalg.svd(a1, full_matrices=False)
    pa2 = u1 @ (u1.T @ a2)
    u, s, vt = np.linalg.svd(a2 - pa2, full_matrices=False)
    t = r - a1.shape[1]
    return pa2 + (u[:, :t] * s[:t]) @ vt[:t]


# --------------------------------------------------------------------------- P1
def test_p1_step0_is_theorem1():
    cfg, a, w1 = cfg1_data()
    res = oracle.swlr(a, w1, cfg.k, cfg.r, iters=0)
    x2 = res.x[:, cfg.k:]
    ref = ghs_by_svd(a[:, :cfg.k], a[:, cfg.k:], cfg.r)
    assert np.linalg.norm(x2 - ref) / np.linalg.norm(ref) < 1e-13
    np.testing.assert_array_equal(res.x[:, :cfg.k], a[:, :cfg.k])


# --------------------------------------------------------------------------- P2
def test_p2_unit_weight_reduces_to_eckart_young():
    """W1 = 1 turns Eq. (5) into Eq. (1): F_N -> sum_{j>r} sigma_j(A)^2
    on 20x30 instances with sigma_r/sigma_{r+1} >= 1.5, k=3, r=5."""
    g = np.random.default_rng(11)
    done = 0
    while done < 4:
        a = g.standard_normal((20, 5)) @ g.standard_normal((5, 30)) + 0.3 * g.standard_normal((20, 30))
        s = np.linalg.svd(a, compute_uv=False)
        if s[4] / s[5] < 1.5:
            continue
        res = oracle.swlr(a, np.ones((20, 3)), 3, 5, iters=2500, eps=1e-13)
        ey = np.sum(s[5:] ** 2)
        assert abs(res.trace[-1]["F"] - ey) / ey < 1e-9
        done += 1


# --------------------------------------------------------------------------- P3
def test_p3_large_weight_approaches_ghs():
    """||X(w) - (A1, GHS(A))|| = O(w^-2) (PAPER.md:67-78 motivation): slope -2."""
    cfg, a, _ = cfg1_data()
    ghs = np.concatenate([a[:, :cfg.k], ghs_by_svd(a[:, :cfg.k], a[:, cfg.k:], cfg.r)], axis=1)
    ws = [1e2, 1e3, 1e4]
    errs = []
    for w in ws:
        res = oracle.swlr(a, np.full((cfg.m, cfg.k), w), cfg.k, cfg.r, iters=60, eps=1e-15)
        errs.append(np.linalg.norm(res.x - ghs) / np.linalg.norm(ghs))
    slope = np.polyfit(np.log10(ws), np.log10(errs), 1)[0]
    assert abs(slope + 2.0) < 0.1, (errs, slope)


# --------------------------------------------------------------------------- P4, P10
@pytest.mark.parametrize("which", ["cfg1", "cfg2", "logw"])
def test_p4_monotone_half_steps_and_p10_rank(which):
    if which == "cfg1":
        cfg, a, w1 = cfg1_data()
        iters = 15
    else:
        cfg = synth.scaled(synth.CONFIGS[2], 30, 40)
        a = synth.make_A(cfg).astype(np.float64)
        w1 = np.full((cfg.m, cfg.k), 100.0)
        if which == "logw":
            w1 = np.exp(np.random.default_rng(5).uniform(0, np.log(1e3), size=(cfg.m, cfg.k)))
        iters = 12
    res = oracle.swlr(a, w1, cfg.k, cfg.r, iters=iters)
    f0 = res.trace[0]["F"]
    slack = 1e-12 * (1 + f0)
    for prev, cur in zip(res.trace[:-1], res.trace[1:]):
        assert cur["F_mid"] <= prev["F"] + slack       # X1 half-step is an exact minimisation
        assert cur["F"] <= cur["F_mid"] + slack        # CD half-step is an exact minimisation
    s = np.linalg.svd(res.x, compute_uv=False)
    assert s[cfg.r] <= 1e-10 * s[0]                  # rank(X_N) <= r


def test_p10_golden_rank_bound():
    g = load("rank_bound.json")
    a = g["A"]
    res = oracle.swlr(a, np.full((4, g["k"]), 3.0), g["k"], g["r"], iters=1)
    assert np.linalg.matrix_rank(a) == g["rank_A"]
    assert res.trace[-1]["F"] < 1e-24
    assert abs(res.trace[-1]["F"] - g["objective_after_one_iteration"]) < 1e-24


# --------------------------------------------------------------------------- P5
def test_p5_theorem2_fixed_point_every_state():
    cfg = synth.scaled(synth.CONFIGS[2], 30, 40)
    a = synth.make_A(cfg).astype(np.float64)
    w1 = np.exp(np.random.default_rng(6).uniform(0, np.log(1e2), size=(cfg.m, cfg.k)))
    a1, a2 = a[:, :cfg.k], a[:, cfg.k:]
    x1 = a1.copy()
    for p in range(6):
        c, d, _ = oracle.cd_step(x1, a2, cfg.r)
        x2 = x1 @ c + d
        ref = ghs_by_svd(x1, a2, cfg.r)            # Theorem 2: GHS applied to X1
        assert np.linalg.norm(x2 - ref) <= 1e-8 * (1 + np.linalg.norm(a2))
        x1 = oracle.x1_step(a1, a2, w1, c, d)


# --------------------------------------------------------------------------- P6
def test_p6_x1_stationarity_and_finite_differences():
    g = np.random.default_rng(7)
    m, n, k, r = 9, 12, 3, 5
    a = g.standard_normal((m, n))
    w1 = g.uniform(5, 10, size=(m, k))
    a1, a2 = a[:, :k], a[:, k:]
    c = g.standard_normal((k, n - k))
    d = g.standard_normal((m, r - k)) @ g.standard_normal((r - k, n - k))
    x1 = oracle.x1_step(a1, a2, w1, c, d)
    # gradient equation after
    grad = -(a1 - x1) * w1 * w1 - (a2 - x1 @ c - d) @ c.T
    assert np.linalg.norm(grad) < 1e-10 * (1 + np.linalg.norm(a))
    # central finite differences of F in X1
    h = 1e-6
    f = lambda z: oracle.objective(a1, a2, w1, z, c, d)
    fd = np.zeros_like(x1)
    for i in range(m):
        for j in range(k):
            e = np.zeros_like(x1)
            e[i, j] = h
            fd[i, j] = (f(x1 + e) - f(x1 - e)) / (2 * h)
    assert np.linalg.norm(fd) < 1e-6 * (1 + f(x1))
    # and it is the unique minimiser: random perturbations increase F
    f0 = f(x1)
    for _ in range(50):
        assert f(x1 + 1e-3 * g.standard_normal(x1.shape)) > f0


# --------------------------------------------------------------------------- P7, P8
def test_p7_scalar_closed_form_golden():
    gd = load("scalar_x1_update.json")
    x = oracle.x1_step(np.array([[gd["a1"]]]), np.array([[gd["a2"]]]), np.array([[gd["w"]]]),
                       np.array([[gd["c"]]]), np.array([[gd["d"]]]))
    assert abs(x[0, 0] - gd["x1"]) < 1e-14


def test_p8_zero_c_gives_a1_and_exact_representability():
    g = np.random.default_rng(8)
    a = g.standard_normal((10, 7))
    w1 = g.uniform(1, 3, size=(10, 2))
    x = oracle.x1_step(a[:, :2], a[:, 2:], w1, np.zeros((2, 5)), g.standard_normal((10, 5)))
    np.testing.assert_allclose(x, a[:, :2], atol=1e-14)
    a = g.standard_normal((12, 4)) @ g.standard_normal((4, 9))      # rank 4 = r
    res = oracle.swlr(a, g.uniform(1, 5, size=(12, 2)), 2, 4, iters=3)
    assert res.trace[-1]["F"] < 1e-20 * np.sum(a * a)


# --------------------------------------------------------------------------- P9
def test_p9_bracketing_by_general_als():
    """the special-weight solution matches a general-weight ALS
    (different parameterisation, X = G H^T) on >= 90% of 20 random instances."""
    g = np.random.default_rng(9)
    agree = 0
    for t in range(20):
        a = g.standard_normal((10, 12))
        w1 = g.uniform(5, 10, size=(10, 2))
        res = oracle.swlr(a, w1, 2, 4, iters=400, eps=1e-14)
        f_s = res.trace[-1]["F"]
        w = np.concatenate([w1, np.ones((10, 10))], axis=1)
        _, f_a = oracle.general_wlra(a, w, 4, restarts=4, inner_iters=400, seed=t)
        if abs(f_s - f_a) <= 1e-6 * (1 + f_s):
            agree += 1
    assert agree >= 18


# --------------------------------------------------------------------------- P11, P12
def test_p11_p12_gram_route_matches_literal():
    """The GPU's map (Cholesky-QR + eigenpairs of S = G_A - M^T C) is the paper's
    (QR + SVD), and F's closed form equals the direct F."""
    for which in (1, 2):
        if which == 1:
            cfg, a, w1 = cfg1_data()
        else:
            cfg = synth.scaled(synth.CONFIGS[2], 30, 40)
            a = synth.make_A(cfg).astype(np.float64)
            w1 = np.full((cfg.m, cfg.k), 100.0)
        a1, a2 = a[:, :cfg.k], a[:, cfg.k:]
        x1 = a1.copy()
        for p in range(4):
            c, d, s = oracle.cd_step(x1, a2, cfg.r)
            st = gram_route.cd_gram(x1, a2, cfg.r)
            assert np.linalg.norm(st["C"] - c) <= 1e-10 * np.linalg.norm(c)
            dg = st["B"] @ st["V"].T
            assert np.linalg.norm(dg - d) <= 1e-9 * np.linalg.norm(d)
            np.testing.assert_allclose(st["lam"], s[: cfg.r - cfg.k] ** 2, rtol=1e-10)
            f_direct = oracle.objective(a1, a2, w1, x1, c, d)
            f_closed = gram_route.objective_closed_form(a1, a2, w1, x1, st)
            assert abs(f_closed - f_direct) <= 1e-9 * f_direct
            x1 = oracle.x1_step(a1, a2, w1, c, d)


def test_step_norm_identity_matches_direct():
    """Error_p from small-side Grams equals ||X_{p+1} - X_p||_F."""
    cfg = synth.scaled(synth.CONFIGS[2], 30, 40)
    a = synth.make_A(cfg).astype(np.float64)
    w1 = np.exp(np.random.default_rng(3).uniform(0, np.log(1e3), size=(cfg.m, cfg.k)))
    a1, a2 = a[:, :cfg.k], a[:, cfg.k:]
    x1 = a1.copy()
    st = gram_route.cd_gram(x1, a2, cfg.r)
    for p in range(5):
        c, d, _ = oracle.cd_step(x1, a2, cfg.r)
        x1n = oracle.x1_step(a1, a2, w1, c, d)
        cn, dn, _ = oracle.cd_step(x1n, a2, cfg.r)
        direct = np.linalg.norm(assemble(x1n, cn, dn) - assemble(x1, c, d)) ** 2
        stn = gram_route.cd_gram(x1n, a2, cfg.r)
        ident = gram_route.step_norm_sq(a2, x1, x1n, st, stn)
        scale = np.sum(assemble(x1, c, d) ** 2)
        assert abs(ident - direct) <= 1e-12 * scale + 1e-6 * direct, (p, ident, direct)
        x1, st = x1n, stn


def test_stopping_rule_or_of_both_tests():
    """PAPER.md:234 / R3: stop on absolute OR relative Error_p below eps."""
    cfg, a, w1 = cfg1_data()
    eps = load("paper_parameters.json")["eps"]
    res = oracle.swlr(a, w1, cfg.k, cfg.r, iters=100, eps=eps)
    assert res.converged
    last = res.trace[-1]
    assert last["step"] < eps or last["rel"] < eps
    for rec in res.trace[1:-1]:
        assert rec["step"] >= eps and rec["rel"] >= eps


def test_invalid_arguments():
    cfg, a, w1 = cfg1_data()
    with pytest.raises(ValueError):
        oracle.swlr(a, w1, cfg.k, cfg.k, iters=1)            # r = k (Theorem 2 needs r > k)
    bad = w1.copy()
    bad[3, 2] = 0.0
    with pytest.raises(ValueError):
        oracle.swlr(a, bad, cfg.k, cfg.r, iters=1)           # W1 > 0
    a0 = a.copy()
    a0[:, 1] = a0[:, 0]
    with pytest.raises(oracle.RankDeficientError):
        oracle.swlr(a0, w1, cfg.k, cfg.r, iters=1)           # rank(A1) < k


def test_r3_relative_error_is_relative_to_the_previous_state():
    """Reading R3: rel_p = ||X_{p+1} - X_p||_F / ||X_p||_F -- the norm of the state
    BEFORE the step, not after.  The states are rebuilt here by separate oracle runs of p and p+1
    iterations, and the case (random X1_0, unit weight) makes ||X_p|| and ||X_{p+1}|| differ by
    far more than the tolerance, so the other denominator fails."""
    g = np.random.default_rng(31)
    a = g.standard_normal((40, 6)) @ g.standard_normal((6, 12)) + 0.1 * g.standard_normal((40, 12))
    w1 = np.ones((40, 3))
    x0 = 5.0 * g.standard_normal((40, 3))           # far from A1: the first steps change ||X|| a lot
    full = oracle.swlr(a, w1, 3, 5, iters=3, x1_0=x0)
    for p in range(3):
        xp = oracle.swlr(a, w1, 3, 5, iters=p, x1_0=x0).x
        xq = oracle.swlr(a, w1, 3, 5, iters=p + 1, x1_0=x0).x
        err = np.linalg.norm(xq - xp)
        before, after = err / np.linalg.norm(xp), err / np.linalg.norm(xq)
        rec = full.trace[p + 1]
        assert abs(rec["step"] - err) <= 1e-12 * err
        assert abs(rec["rel"] - before) <= 1e-12 * before
        if p == 0:
            assert abs(after - before) > 1e-3 * before   # the two readings are distinguishable
