"""Brute-force general weighted low-rank approximation -- TEST INFRASTRUCTURE ONLY.

Solves Eq. (6), min ||(A - X) . W||_F^2 over rank(X) <= r, for
small matrices by multi-start alternating weighted least squares on X = G H^T
(SPEC.md:350-358).  It deliberately uses a different parameterisation from sWLR's
(X1, C, D), so agreement with ``oracle.swlr`` on the special weight W = (W1 1) is
evidence, not tautology (pin P9).
"""
from __future__ import annotations

import numpy as np


def _wls_rows(a, w, h, ridge):
    """Row-wise weighted LS: for each i, g_i = argmin sum_j w_ij^2 (a_ij - g_i . h_j)^2."""
    m = a.shape[0]
    r = h.shape[1]
    g = np.empty((m, r))
    for i in range(m):
        w2 = w[i] ** 2
        lhs = (h * w2[:, None]).T @ h + ridge * np.eye(r)
        rhs = (h * w2[:, None]).T @ a[i]
        g[i] = np.linalg.solve(lhs, rhs)
    return g


def general_wlra(a, w, r, restarts=10, inner_iters=500, tol=1e-13, seed=0):
    """Best objective over ``restarts`` alternating-minimisation runs.
    Returns (X, objective)."""
    a = np.asarray(a, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    m, n = a.shape
    rng = np.random.default_rng(seed)
    best = (None, np.inf)
    for s in range(restarts):
        if s == 0:   # one start from the unweighted truncated SVD
            u, sv, vt = np.linalg.svd(a, full_matrices=False)
            h = vt[:r].T * sv[:r]
        else:
            h = rng.standard_normal((n, r))
        prev = np.inf
        for _ in range(inner_iters):
            g = _wls_rows(a, w, h, 1e-12)
            h = _wls_rows(a.T, w.T, g, 1e-12)
            f = float(np.sum(((a - g @ h.T) * w) ** 2))
            if prev - f <= tol * (1.0 + f):
                break
            prev = f
        if f < best[1]:
            best = (g @ h.T, f)
    return best
