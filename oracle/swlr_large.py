"""Algorithm 1 for large m (m >= 1e5) -- TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The same iteration as ``oracle.swlr.swlr`` (readings R1-R16), restated so
that BASELINE.json config 5 (m = 921 600, n = 1000, k = 100, r = 110) fits the host:

* CD half-step (Algorithm 1 lines 4-6):
  (X1)_p = Q_p R_p (Householder QR), C_p = R_p^{-1} Q_p^T A2, P = (I - Q_p Q_p^T) A2.
  The top r-k singular triplets of P come from the symmetric eigenproblem of the explicit
  fp64 Gram P^T P (eigenvalues sigma^2, eigenvectors = right singular vectors V), the reading
  SURVEY.md §8(c) prescribes for m >= 1e5 (reading R22).  D_p = U (Sigma_p)_{r-k} V^T
  is kept in its product form D_p = B_p V_t^T with B_p = U_t Sigma_t = P V_t (m x (r-k)) -- the
  same matrix, never assembled (7 GB at config 5).
* X1 half-step (Algorithm 1 lines 7-9; Eq. (9) and the row formula
  PAPER.md:184-196): E_p = A1 . W1 . W1 + (A2 - D_p) C_p^T, then
  X1(i,:) = E(i,:) (diag(W1(i,:)^2) + C_p C_p^T)^{-1} row by row (R4: row order irrelevant, so
  row chunks run on host threads; R8: the inverse is applied as a linear solve).
* F_p (R11) and Error_p = ||X_{p+1} - X_p||_F (R3) are sums of per-row terms,
  evaluated over row chunks.

Only the SVD -> eigh(P^T P) substitution and the factored D differ from the literal oracle;
``tests/test_oracle_large.py`` pins this module against ``oracle.swlr`` (which is itself pinned
by P1-P12) on inputs where both run, and checks the invariants (monotone half-steps, Theorem-2
fixed point) directly.  A is accepted in fp32 (the fp32 configs' data, R12) and upcast to fp64
chunk by chunk, which is exact.
"""
from __future__ import annotations

import concurrent.futures as cf
import dataclasses
from typing import List, Optional

import numpy as np
import scipy.linalg

from .swlr import qr_thin

CHUNK = 16384


def _chunks(m: int, chunk: int = CHUNK):
    return [(i0, min(i0 + chunk, m)) for i0 in range(0, m, chunk)]


def _w1rows(w1, w_const, i0, i1, k):
    if w1 is None:
        return np.full((i1 - i0, k), float(w_const))
    return np.asarray(w1[i0:i1], dtype=np.float64)


@dataclasses.dataclass
class CDState:
    """(C_p, D_p) of one canonical state with D_p = B V^T."""
    c: np.ndarray          # k x (n-k)
    b: np.ndarray          # m x (r-k)  = U_t Sigma_t
    vt: np.ndarray         # (r-k) x (n-k)
    sigma: np.ndarray      # singular values of P (descending, all n-k of them)


def cd_step_gram(x1: np.ndarray, a: np.ndarray, k: int, r: int, pool) -> CDState:
    """(C_p, D_p) = argmin F((X1)_p, C, D), PAPER.md:143-165 / Algorithm 1 lines 4-6, with the
    singular triplets of P = (I - QQ^T) A2 from eigh(P^T P) (R22)."""
    m, n = a.shape
    if r <= k:
        raise ValueError("cd_step_gram: Theorem 2 needs r > k (PAPER.md:94; R7)")
    q, rr = qr_thin(x1)                                           # (X1)_p = Q_p R_p
    parts = list(pool.map(lambda c: q[c[0]:c[1]].T @ np.asarray(a[c[0]:c[1], k:], np.float64),
                          _chunks(m)))
    qta2 = np.sum(parts, axis=0)                                  # Q^T A2
    c = scipy.linalg.solve_triangular(rr, qta2, lower=False)      # C_p = R^{-1} Q^T A2

    def ptp(ch):
        i0, i1 = ch
        p = np.asarray(a[i0:i1, k:], np.float64) - q[i0:i1] @ qta2   # rows of (I - QQ^T) A2
        return p.T @ p
    g = np.sum(list(pool.map(ptp, _chunks(m))), axis=0)
    g = 0.5 * (g + g.T)
    lam, vec = np.linalg.eigh(g)                                  # ascending
    lam, vec = lam[::-1], vec[:, ::-1]
    t = r - k
    vt = np.ascontiguousarray(vec[:, :t].T)                       # V_t^T

    def bpart(ch):
        i0, i1 = ch
        p = np.asarray(a[i0:i1, k:], np.float64) - q[i0:i1] @ qta2
        return p @ vt.T                                           # U_t Sigma_t = P V_t
    b = np.concatenate(list(pool.map(bpart, _chunks(m))), axis=0)
    sigma = np.sqrt(np.maximum(lam, 0.0))
    return CDState(c=c, b=b, vt=vt, sigma=sigma)


def x1_step_rows(a, w1, w_const, k, st: CDState, pool) -> np.ndarray:
    """(X1)_{p+1}, Eq. (9) / PAPER.md:194-196 (Algorithm 1 lines 7-9), rows in parallel (R4)."""
    m = a.shape[0]
    c = st.c
    cct = c @ c.T
    out = np.empty((m, k))
    idx = np.arange(k)

    def rows(ch):
        i0, i1 = ch
        ar = np.asarray(a[i0:i1], np.float64)
        w = _w1rows(w1, w_const, i0, i1, k)
        d = st.b[i0:i1] @ st.vt                                   # rows of D_p
        e = ar[:, :k] * w * w + (ar[:, k:] - d) @ c.T             # rows of E_p
        kmat = np.broadcast_to(cct, (i1 - i0, k, k)).copy()
        kmat[:, idx, idx] += w * w                                # diag(W1(i,:)^2) + C C^T
        out[i0:i1] = np.linalg.solve(kmat, e[:, :, None])[:, :, 0]
    list(pool.map(rows, _chunks(m, 4096)))
    return out


def objective_rows(a, w1, w_const, k, x1, st: CDState, pool) -> float:
    """F(X1, C, D) = ||(A1 - X1) . W1||^2 + ||A2 - X1 C - D||^2."""
    def part(ch):
        i0, i1 = ch
        ar = np.asarray(a[i0:i1], np.float64)
        w = _w1rows(w1, w_const, i0, i1, k)
        fw = np.sum(((ar[:, :k] - x1[i0:i1]) * w) ** 2)
        res = ar[:, k:] - x1[i0:i1] @ st.c - st.b[i0:i1] @ st.vt
        return fw + np.sum(res * res)
    return float(np.sum(list(pool.map(part, _chunks(m=a.shape[0])))))


def step_sq_rows(x1n, stn: CDState, x1, st: CDState, pool):
    """||X_{p+1} - X_p||_F^2 and ||X_p||_F^2 with X_p = (X1_p, X1_p C_p + D_p)."""
    def part(ch):
        i0, i1 = ch
        x2n = x1n[i0:i1] @ stn.c + stn.b[i0:i1] @ stn.vt
        x2 = x1[i0:i1] @ st.c + st.b[i0:i1] @ st.vt
        d1 = x1n[i0:i1] - x1[i0:i1]
        d2 = x2n - x2
        return np.array([np.sum(d1 * d1) + np.sum(d2 * d2),
                         np.sum(x1[i0:i1] ** 2) + np.sum(x2 * x2)])
    s = np.sum(list(pool.map(part, _chunks(x1.shape[0]))), axis=0)
    return float(s[0]), float(s[1])


@dataclasses.dataclass
class LargeResult:
    x1: np.ndarray
    st: CDState
    trace: List[dict]
    converged: bool

    def x_rows(self, rows: np.ndarray) -> np.ndarray:
        """Rows of X_N = (X1_N, X1_N C_N + D_N) (R1)."""
        x1 = self.x1[rows]
        return np.concatenate([x1, x1 @ self.st.c + self.st.b[rows] @ self.st.vt], axis=1)


def swlr_large(a: np.ndarray, w1: Optional[np.ndarray], k: int, r: int, iters: int,
               w_const: float = 1.0, x1_0: Optional[np.ndarray] = None, eps: float = 0.0,
               threads: int = 8, log=None) -> LargeResult:
    """Algorithm 1 with the same state, trace records and stopping rule as
    ``oracle.swlr.swlr``; ``w1`` = None means W1 is uniform with value ``w_const``."""
    m, n = a.shape
    if not (1 <= k < n) or not (k < r <= min(m, n)):
        raise ValueError("need 1 <= k < n and k < r <= min(m, n)")
    if w1 is None:
        if not w_const > 0:
            raise ValueError("W1 must be > 0 (PAPER.md:94; R16)")
    elif w1.shape != (m, k) or not np.all(w1 > 0):
        raise ValueError("W1 must be m x k with entries > 0 (PAPER.md:94; R16)")
    t = r - k
    with cf.ThreadPoolExecutor(threads) as pool:
        x1 = (np.asarray(a[:, :k], np.float64).copy() if x1_0 is None
              else np.asarray(x1_0, np.float64).copy())
        st = cd_step_gram(x1, a, k, r, pool)

        def sig(sv, j):
            return float(sv[j]) if j < sv.size else 0.0
        trace = [dict(p=0, F=objective_rows(a, w1, w_const, k, x1, st, pool),
                      sig_t=sig(st.sigma, t - 1), sig_t1=sig(st.sigma, t))]
        converged = False
        for p in range(iters):
            x1n = x1_step_rows(a, w1, w_const, k, st, pool)                  # lines 7-9
            f_mid = objective_rows(a, w1, w_const, k, x1n, st, pool)
            stn = cd_step_gram(x1n, a, k, r, pool)                           # lines 4-6
            e2, xs2 = step_sq_rows(x1n, stn, x1, st, pool)
            err = float(np.sqrt(e2))
            rel = err / float(np.sqrt(xs2))
            trace.append(dict(p=p + 1, F=objective_rows(a, w1, w_const, k, x1n, stn, pool),
                              F_mid=f_mid, step=err, rel=rel, sig_t=sig(stn.sigma, t - 1),
                              sig_t1=sig(stn.sigma, t)))
            if log is not None:
                log(trace[-1])
            x1, st = x1n, stn
            if eps > 0.0 and (err < eps or rel < eps):
                converged = True
                break
    return LargeResult(x1=x1, st=st, trace=trace, converged=converged)
