"""the factorised WLR iteration as a one-sweep block ALS on
(X1, C, B, D), X2 = X1 C + B D.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md contrasts sWLR with the factorisation-based WLR of its refs [duttali, duttali_cvpr]
("the authors proposed an algorithm WLR ...", "Our new algorithm is not
based on matrix factorization to address the rank constraint", and the X1 update written with
(C_p, B_p) at PAPER.md:188).  The factorised iteration is not spelled out in PAPER.md; the
reading used here is DESIGN.md R21:

* state (X1, C, B, D): X1 m x k, C k x (n-k), B m x (r-k), D (r-k) x (n-k);
* p = 0 is the GHS point (Theorem 1): X1_0 = A1, C_0 = A1^+ A2 and
  B_0 D_0 = H_{r-k}(P^perp_{A1} A2) split as B_0 = U Sigma, D_0 = V^T (thin SVD);
* one iteration p -> p+1 is one sweep of exact block minimisations of
  F(X1, C, B, D) = ||(A1 - X1) . W1||_F^2 + ||A2 - X1 C - B D||_F^2:
    1. X1 <- argmin_X1 F          the row formula of PAPER.md:184-196 with D_p := B_p D_p
    2. C  <- argmin_C  F          least squares  X1 C ~ A2 - B_p D_p
    3. B  <- argmin_B  F          least squares  B D_p ~ A2 - X1 C
    4. D  <- argmin_D  F          least squares  B D ~ A2 - X1 C
  (the order of SURVEY.md §8(f3): B = (A2 - X1 C) D^T (D D^T)^{-1}, D = (B^T B)^{-1} B^T (A2 - X1 C)).
Every block step is the exact minimiser of a convex quadratic in that block, so F is
non-increasing along the sweep (a pin).  Unlike sWLR's (C, D) step (Theorem 2), the (C, B, D)
sweep is not the joint minimiser over (C, D) for fixed X1, so the iterates differ from sWLR's.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np

from .swlr import qr_thin, svd_thin, x1_step


def objective4(a1, a2, w1, x1, c, b, d) -> float:
    """F(X1, C, B, D) = ||(A1 - X1) . W1||_F^2 + ||A2 - X1 C - B D||_F^2 (PAPER.md:141-142 with
    the rank-(r-k) term D of Eq. (8) factorised as B D)."""
    return float(np.sum(((a1 - x1) * w1) ** 2) + np.sum((a2 - x1 @ c - b @ d) ** 2))


def ghs_factors(a1, a2, r):
    """GHS start (Theorem 1) in factorised form: C_0 = R^{-1} Q^T A2 with
    A1 = Q R, and the rank-(r-k) truncated SVD of (I - Q Q^T) A2 = U Sigma V^T split as
    B_0 = U_{r-k} Sigma_{r-k}, D_0 = V_{r-k}^T."""
    k = a1.shape[1]
    t = r - k
    q, rr = qr_thin(a1)
    qta2 = q.T @ a2
    c = np.linalg.solve(rr, qta2)
    u, s, vt = svd_thin(a2 - q @ qta2)
    return c, u[:, :t] * s[:t], vt[:t].copy()


def c_step(x1, a2, b, d):
    """C = argmin_C ||A2 - B D - X1 C||_F (step 2 of R21): least squares (LAPACK gelsd)."""
    return np.linalg.lstsq(x1, a2 - b @ d, rcond=None)[0]


def b_step(x1, c, a2, d):
    """B = argmin_B ||(A2 - X1 C) - B D||_F = (A2 - X1 C) D^T (D D^T)^{-1} (step 3 of R21),
    as the least-squares problem D^T B^T ~ (A2 - X1 C)^T."""
    return np.linalg.lstsq(d.T, (a2 - x1 @ c).T, rcond=None)[0].T


def d_step(x1, c, a2, b):
    """D = argmin_D ||(A2 - X1 C) - B D||_F = (B^T B)^{-1} B^T (A2 - X1 C) (step 4 of R21)."""
    return np.linalg.lstsq(b, a2 - x1 @ c, rcond=None)[0]


@dataclasses.dataclass
class BlockAlsResult:
    x1: np.ndarray
    c: np.ndarray
    b: np.ndarray
    d: np.ndarray
    trace: List[dict]          # per state p: F_p, and for p >= 1 the F after each sub-step


def block_als(a: np.ndarray, w1: np.ndarray, k: int, r: int, iters: int,
              x1_0: Optional[np.ndarray] = None) -> BlockAlsResult:
    """R21 block ALS from the GHS point (or from a given X1_0 with (C, B, D) from the
    factorised GHS formulas applied to X1_0), ``iters`` sweeps, in fp64."""
    a = np.asarray(a, dtype=np.float64)
    w1 = np.asarray(w1, dtype=np.float64)
    m, n = a.shape
    if not (1 <= k < n) or not (k < r <= min(m, n)):
        raise ValueError("need 1 <= k < n and k < r <= min(m, n)")
    if w1.shape != (m, k) or not np.all(w1 > 0):
        raise ValueError("W1 must be m x k with entries > 0 (PAPER.md:94)")
    a1, a2 = a[:, :k], a[:, k:]
    x1 = a1.copy() if x1_0 is None else np.asarray(x1_0, dtype=np.float64).copy()
    c, b, d = ghs_factors(x1, a2, r)
    trace = [dict(p=0, F=objective4(a1, a2, w1, x1, c, b, d))]
    for p in range(iters):
        x1 = x1_step(a1, a2, w1, c, b @ d)                   # 1. PAPER.md:184-196, D_p = B_p D_p
        f1 = objective4(a1, a2, w1, x1, c, b, d)
        c = c_step(x1, a2, b, d)                             # 2.
        f2 = objective4(a1, a2, w1, x1, c, b, d)
        b = b_step(x1, c, a2, d)                             # 3.
        f3 = objective4(a1, a2, w1, x1, c, b, d)
        d = d_step(x1, c, a2, b)                             # 4.
        f4 = objective4(a1, a2, w1, x1, c, b, d)
        trace.append(dict(p=p + 1, F=f4, F_x1=f1, F_c=f2, F_b=f3))
    return BlockAlsResult(x1=x1, c=c, b=b, d=d, trace=trace)
