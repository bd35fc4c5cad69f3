"""Literal fp64 transcription of the sWLR algorithm -- TEST INFRASTRUCTURE ONLY.

See ``oracle/__init__.py`` for the import rule.  Every function cites the PAPER.md
lines (and section / equation / algorithm line) it follows; "Rn" refers to the
readings listed in DESIGN.md "Readings of the paper".

Notation: A = (A1 A2) is m x n, A1 = first k columns,
W = (W1 1) with W1 > 0 (m x k), X = (X1 X2) with X2 = X1 C + D, rank(D) <= r-k.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np
import scipy.linalg

RANK_TOL = 1e-12          # SPEC.md:64 / SPEC.md:104: |R_ii| < 1e-12 * ||X1||_F => deficient


class RankDeficientError(np.linalg.LinAlgError):
    """X1 is numerically rank deficient (PAPER.md:133 assumes r(X1) = k; R6)."""

    def __init__(self, index: int):
        super().__init__(f"rank-deficient: |R[{index},{index}]| below tolerance")
        self.index = index


# ----------------------------------------------------------------- dense primitives
def svd_thin(a: np.ndarray):
    """Thin SVD a = U diag(s) Vt ("A = U Sigma V^T is a SVD of A").
    LAPACK gesdd via numpy; singular values non-increasing."""
    a = np.asarray(a, dtype=np.float64)
    if not np.all(np.isfinite(a)):
        raise ValueError("svd_thin: non-finite input")
    return np.linalg.svd(a, full_matrices=False)


def qr_thin(x: np.ndarray):
    """Thin Householder QR x = Q R ("(X1)_p = Q_p R_p"), with the
    rank test of SPEC.md:64 (R6)."""
    x = np.asarray(x, dtype=np.float64)
    q, r = np.linalg.qr(x, mode="reduced")
    nrm = np.linalg.norm(x)
    d = np.abs(np.diag(r))
    bad = np.nonzero(d < RANK_TOL * max(nrm, np.finfo(float).tiny))[0]
    if bad.size:
        raise RankDeficientError(int(bad[0]))
    return q, r


def hard_threshold(a: np.ndarray, rank: int) -> np.ndarray:
    """H_rank(a) = U Sigma_rank V^T: keep the largest ``rank`` singular values and
    replace the others by 0 (Eq. (2)).  Ties at the cut keep the
    first ``rank`` in LAPACK order (R9)."""
    u, s, vt = svd_thin(a)
    rank = max(0, min(rank, s.size))
    return (u[:, :rank] * s[:rank]) @ vt[:rank]


def pca_truncate(a: np.ndarray, r: int) -> np.ndarray:
    """Solution of the PCA problem Eq. (1) given by Eq. (2)."""
    return hard_threshold(a, r)


def ghs_solve(a1: np.ndarray, a2: np.ndarray, r: int) -> np.ndarray:
    """Golub-Hoffman-Stewart, Theorem 1 / Eq. (4):
    A~2 = P_{A1}(A2) + H_{r-k}(P^perp_{A1}(A2)), k = r(A1) <= r.
    The column-space basis comes from QR of A1; a numerically
    rank-deficient A1 raises (R13)."""
    k = a1.shape[1]
    if r < k:
        raise ValueError("ghs_solve: Theorem 1 needs r >= k")
    q, _ = qr_thin(a1)
    pa2 = q @ (q.T @ a2)                       # P_{A1}(A2)
    return pa2 + hard_threshold(a2 - pa2, r - k)


def objective(a1, a2, w1, x1, c, d) -> float:
    """F(X1, C, D) = ||(A1 - X1) . W1||_F^2 + ||A2 - X1 C - D||_F^2
    (objective of Eq. (8))."""
    fw = np.sum(((a1 - x1) * w1) ** 2)
    fu = np.sum((a2 - x1 @ c - d) ** 2)
    return float(fw + fu)


# ------------------------------------------------------------------ the two half-steps
def cd_step(x1: np.ndarray, a2: np.ndarray, r: int):
    """(C_p, D_p) = argmin_{C,D} F((X1)_p, C, D), PAPER.md:143-165 and Algorithm 1
    lines 4-6:
        (X1)_p = Q_p R_p;   (I - Q_p Q_p^T) A2 = U_p Sigma_p V_p^T;
        C_p = R_p^{-1} Q_p^T A2;   D_p = U_p (Sigma_p)_{r-k} V_p^T.
    Returns (C, D, sigma) with sigma the singular values of (I - QQ^T) A2."""
    k = x1.shape[1]
    if r <= k:
        raise ValueError("cd_step: Theorem 2 needs r > k (PAPER.md:94; R7)")
    q, rr = qr_thin(x1)
    qta2 = q.T @ a2
    c = scipy.linalg.solve_triangular(rr, qta2, lower=False)       # R^{-1} Q^T A2
    p = a2 - q @ qta2                                              # (I - QQ^T) A2
    u, s, vt = svd_thin(p)
    t = r - k
    d = (u[:, :t] * s[:t]) @ vt[:t]                                # U (Sigma)_{r-k} V^T
    return c, d, s


def x1_step(a1, a2, w1, c, d, chunk: int = 4096) -> np.ndarray:
    """(X1)_{p+1} = argmin_{X1} F(X1, C_p, D_p), Eq. (9) and the row formula
    (PAPER.md:184-196), Algorithm 1 lines 7-9:
        E_p = A1 . W1 . W1 + (A2 - D_p) C_p^T
        X1(i,:) = E(i,:) (diag(W1(i,1)^2 ... W1(i,k)^2) + C_p C_p^T)^{-1}   for i = 1..m.
    The inverse is applied as a linear solve with the (symmetric) row matrix (R8);
    rows are independent given (C_p, D_p), so their order is irrelevant (R4)."""
    e = a1 * w1 * w1 + (a2 - d) @ c.T
    cct = c @ c.T
    m, k = a1.shape
    x1 = np.empty((m, k))
    for i0 in range(0, m, chunk):
        i1 = min(i0 + chunk, m)
        kmat = np.broadcast_to(cct, (i1 - i0, k, k)).copy()
        idx = np.arange(k)
        kmat[:, idx, idx] += w1[i0:i1] ** 2
        # x K = e  <=>  K x^T = e^T  (K symmetric)
        x1[i0:i1] = np.linalg.solve(kmat, e[i0:i1, :, None])[:, :, 0]
    return x1


# -------------------------------------------------------------------- Algorithm 1
@dataclasses.dataclass
class SwlrResult:
    x1: np.ndarray            # (X1)_N
    c: np.ndarray             # C_N
    d: np.ndarray             # D_N
    x: np.ndarray             # X_N = ((X1)_N, (X1)_N C_N + D_N)
    trace: List[dict]         # one record per canonical state p = 0..N
    converged: bool


def assemble(x1, c, d) -> np.ndarray:
    """X_p = ((X1)_p, (X1)_p C_p + D_p)  (R1)."""
    return np.concatenate([x1, x1 @ c + d], axis=1)


def swlr(a: np.ndarray, w1: np.ndarray, k: int, r: int, iters: int,
         x1_0: Optional[np.ndarray] = None, eps: float = 0.0) -> SwlrResult:
    """Algorithm 1, "sWLR Algorithm", in fp64.

    * Input A = (A1 A2), W = (W1 1) (line 1); W1 given as an m x k array.
    * Initialise (X1)_0 (line 2): A1 (GHS start, R5) unless ``x1_0`` is given.
    * Canonical state after iteration p (R1): X_p = ((X1)_p,
      (X1)_p C_p + D_p) with (C_p, D_p) = cd_step((X1)_p); "N iterations" = N X1
      half-steps and N+1 CD half-steps.
    * Stopping (R3): Error_p = ||X_{p+1} - X_p||_F; stop when
      Error_p < eps or Error_p / ||X_p||_F < eps (ORed), or after ``iters``.
      eps = 0 runs exactly ``iters`` iterations.
    Trace record p holds F_p = F((X1)_p, C_p, D_p) (R11); records p >= 1 also hold
    F_mid = F((X1)_p, C_{p-1}, D_{p-1}), step = Error_{p-1}, rel = step/||X_{p-1}||,
    and sigma_{r-k}, sigma_{r-k+1} of P^perp A2 at state p.
    """
    a = np.asarray(a, dtype=np.float64)
    w1 = np.asarray(w1, dtype=np.float64)
    m, n = a.shape
    if not (1 <= k < n) or not (k < r <= min(m, n)):
        raise ValueError("need 1 <= k < n and k < r <= min(m, n)")
    if w1.shape != (m, k) or not np.all(w1 > 0):
        raise ValueError("W1 must be m x k with entries > 0 (PAPER.md:94; R16)")
    a1, a2 = a[:, :k], a[:, k:]
    x1 = a1.copy() if x1_0 is None else np.asarray(x1_0, dtype=np.float64).copy()
    c, d, s = cd_step(x1, a2, r)
    x = assemble(x1, c, d)
    t = r - k

    def sig(sv, j):
        return float(sv[j]) if j < sv.size else 0.0

    trace = [dict(p=0, F=objective(a1, a2, w1, x1, c, d), sig_t=sig(s, t - 1), sig_t1=sig(s, t))]
    converged = False
    for p in range(iters):
        x1n = x1_step(a1, a2, w1, c, d)                       # lines 7-9
        f_mid = objective(a1, a2, w1, x1n, c, d)
        cn, dn, sn = cd_step(x1n, a2, r)                      # lines 4-6 at p+1
        xn = assemble(x1n, cn, dn)
        err = float(np.linalg.norm(xn - x))
        rel = err / float(np.linalg.norm(x))
        trace.append(dict(p=p + 1, F=objective(a1, a2, w1, x1n, cn, dn), F_mid=f_mid,
                          step=err, rel=rel, sig_t=sig(sn, t - 1), sig_t1=sig(sn, t)))
        x1, c, d, x = x1n, cn, dn, xn
        if eps > 0.0 and (err < eps or rel < eps):
            converged = True
            break
    return SwlrResult(x1=x1, c=c, d=d, x=x, trace=trace, converged=converged)
