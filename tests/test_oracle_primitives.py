"""Pins for the oracle's dense primitives (CPU).  SPEC.md:97-101 invariants,
SPEC.md:57-95 examples, and the hand-computed fixtures in tests/golden/."""
import numpy as np
import pytest

import oracle
from tests.golden_io import load

pytestmark = pytest.mark.filterwarnings("ignore")


def rng(seed=0):
    return np.random.default_rng(seed)


def test_golden_eckart_young_diag():
    g = load("eckart_young_diag.json")
    h = oracle.hard_threshold(g["A"], g["r"])
    np.testing.assert_allclose(h, g["H_r"], atol=1e-14)
    assert abs(np.sum((g["A"] - h) ** 2) - g["objective"]) < 1e-13


def test_golden_ghs_hand():
    g = load("ghs_hand.json")
    k, r = g["k"], g["r"]
    a2t = oracle.ghs_solve(g["A"][:, :k], g["A"][:, k:], r)
    np.testing.assert_allclose(a2t, g["A2_tilde"], atol=1e-13)
    assert abs(np.sum((g["A"][:, k:] - a2t) ** 2) - g["objective"]) < 1e-12


def test_svd_invariants_200_matrices():
    """SPEC.md:98 reconstruction <= 1e-8, orthonormal factors."""
    g = rng(1)
    for t in range(200):
        m, n = g.integers(1, 9, size=2)
        a = g.standard_normal((m, n)) * 10.0 ** g.uniform(-3, 3)
        u, s, vt = oracle.svd_thin(a)
        assert np.all(np.diff(s) <= 1e-12 * max(1, s[0])) and np.all(s >= 0)
        assert np.linalg.norm(u * s @ vt - a) <= 1e-8 * max(1.0, np.linalg.norm(a))
        np.testing.assert_allclose(u.T @ u, np.eye(u.shape[1]), atol=1e-10)
        np.testing.assert_allclose(vt @ vt.T, np.eye(vt.shape[0]), atol=1e-10)


def test_svd_trivial_examples():
    s = oracle.svd_thin(np.diag([3.0, 2.0]))[1]
    np.testing.assert_allclose(s, [3.0, 2.0])
    s = oracle.svd_thin(np.zeros((3, 2)))[1]
    np.testing.assert_allclose(s, [0.0, 0.0])


def test_qr_examples_and_rank_error():
    q, r = oracle.qr_thin(np.array([[3.0], [4.0]]))
    assert abs(abs(r[0, 0]) - 5.0) < 1e-14
    np.testing.assert_allclose(np.abs(q[:, 0]), [0.6, 0.8], atol=1e-15)
    a = rng(2).standard_normal((6, 3))
    q, r = oracle.qr_thin(a)
    np.testing.assert_allclose(q.T @ q, np.eye(3), atol=1e-12)
    np.testing.assert_allclose(q @ r, a, atol=1e-12)
    b = np.column_stack([a[:, 0], a[:, 1], a[:, 0] + a[:, 1]])   # rank 2
    with pytest.raises(oracle.RankDeficientError) as ei:
        oracle.qr_thin(b)
    assert ei.value.index == 2


def test_hard_threshold_properties():
    g = rng(3)
    a = g.standard_normal((5, 5))
    h2 = oracle.hard_threshold(a, 2)
    assert np.linalg.matrix_rank(h2) == 2
    np.testing.assert_allclose(oracle.hard_threshold(a, 5), a, atol=1e-12)
    assert np.all(oracle.hard_threshold(a, 0) == 0)
    # scale equivariance
    np.testing.assert_allclose(oracle.hard_threshold(3.7 * a, 2), 3.7 * h2, rtol=1e-10, atol=1e-12)
    # Eckart-Young optimality vs 1000 random rank-2 competitors
    best = np.linalg.norm(a - h2)
    for _ in range(1000):
        y = g.standard_normal((5, 2)) @ g.standard_normal((2, 5))
        assert best <= np.linalg.norm(a - y) + 1e-12
    # objective equals the tail of the spectrum
    b = g.standard_normal((8, 6))
    s = np.linalg.svd(b, compute_uv=False)
    assert abs(np.sum((b - oracle.pca_truncate(b, 3)) ** 2) - np.sum(s[3:] ** 2)) < 1e-10


def test_projector_decomposition():
    """P(b) + Pperp(b) = b and <P b, Pperp b> = 0, via qr_thin's basis."""
    g = rng(4)
    q, _ = oracle.qr_thin(g.standard_normal((7, 3)))
    b = g.standard_normal((7, 4))
    pb = q @ (q.T @ b)
    np.testing.assert_allclose(q @ (q.T @ pb), pb, atol=1e-12)
    assert abs(np.sum(pb * (b - pb))) < 1e-12


def test_ghs_in_colspace_and_dominance():
    g = rng(5)
    a1 = g.standard_normal((6, 2))
    a2 = a1 @ g.standard_normal((2, 6))              # A2 in colspace(A1): A~2 = A2
    np.testing.assert_allclose(oracle.ghs_solve(a1, a2, 4), a2, atol=1e-12)
    a2 = g.standard_normal((6, 6))
    best = np.linalg.norm(a2 - oracle.ghs_solve(a1, a2, 4))
    for _ in range(500):   # any X2 with rank(A1 X2) <= 4 is A1 C + D with rank(D) <= 2
        x2 = a1 @ g.standard_normal((2, 6)) + g.standard_normal((6, 2)) @ g.standard_normal((2, 6))
        assert best <= np.linalg.norm(a2 - x2) + 1e-12


def test_golden_objective_hand():
    g = load("objective_hand.json")
    f = oracle.objective(g["A1"], g["A2"], g["W1"], g["X1"], g["C"], g["D"])
    assert abs(f - g["F"]) < 1e-14
    # W1 = 1 reduces to the unweighted residual
    ones = np.ones_like(g["W1"])
    x = np.concatenate([g["X1"], g["X1"] @ g["C"] + g["D"]], axis=1)
    a = np.concatenate([g["A1"], g["A2"]], axis=1)
    assert abs(oracle.objective(g["A1"], g["A2"], ones, g["X1"], g["C"], g["D"]) - np.sum((a - x) ** 2)) < 1e-14


def test_x1_step_chunking_is_row_independent():
    """Rows are independent given (C, D) (R4): chunk size cannot change the result."""
    g = np.random.default_rng(12)
    a = g.standard_normal((50, 9))
    w1 = g.uniform(1, 10, size=(50, 3))
    c = g.standard_normal((3, 6))
    d = g.standard_normal((50, 2)) @ g.standard_normal((2, 6))
    x_all = oracle.x1_step(a[:, :3], a[:, 3:], w1, c, d)
    x_chk = oracle.x1_step(a[:, :3], a[:, 3:], w1, c, d, chunk=7)
    np.testing.assert_allclose(x_chk, x_all, rtol=0, atol=1e-13)
    # row i alone gives the same row
    x_5 = oracle.x1_step(a[5:6, :3], a[5:6, 3:], w1[5:6], c, d[5:6])
    np.testing.assert_allclose(x_5[0], x_all[5], atol=1e-13)
