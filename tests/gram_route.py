"""Test-only fp64 restatement of the *Gram route* the CUDA path takes.

It is NOT the oracle: it exists to pin, against the literal oracle, that the
mathematical map the GPU implements is the paper's (pins P11 and P12, and the
small-side step-norm identity of SURVEY.md §8(a) a5).  It shares no code with the
CUDA path (which is C++/CUDA) and is not imported by it.

    G = X1^T X1,  M = X1^T A2,  G_A = A2^T A2
    C = G^{-1} M                              (= R^{-1} Q^T A2)
    S = G_A - M^T C = A2^T P^perp A2          (right Gram of P^perp A2)
    (lambda, V) = top r-k eigenpairs of S      (lambda = sigma^2, V = right sing. vectors)
    D = (A2 - X1 C) V V^T                      (= U Sigma_{r-k} V^T)
    F = sum W1^2 (A1 - X1)^2 + ||A2||^2 - <M, C> - sum(lambda)
"""
import numpy as np


def cd_gram(x1, a2, r):
    k = x1.shape[1]
    g = x1.T @ x1
    m = x1.T @ a2
    l = np.linalg.cholesky(g)
    c = np.linalg.solve(l.T, np.linalg.solve(l, m))
    s = a2.T @ a2 - m.T @ c
    lam, vec = np.linalg.eigh(s)
    lam, vec = lam[::-1][: r - k], vec[:, ::-1][:, : r - k]
    return dict(G=g, M=m, C=c, lam=lam, V=vec, B=(a2 - x1 @ c) @ vec)


def objective_closed_form(a1, a2, w1, x1, st):
    fw = np.sum(((a1 - x1) * w1) ** 2)
    return fw + np.sum(a2 * a2) - np.sum(st["M"] * st["C"]) - np.sum(st["lam"])


def step_norm_sq(a2, x1, x1n, st, stn):
    """||X_{p+1} - X_p||_F^2 from small-side quantities only.
    With P_V = V V^T and X2 = X1 C (I - P_V) + A2 P_V:
      <X2', X2> = tr[(I-P')C'^T H C (I-P)] + tr[(I-P') M'^T... ] etc., H = X1'^T X1."""
    ga = a2.T @ a2
    c, v, m = st["C"], st["V"], st["M"]
    cn, vn, mn = stn["C"], stn["V"], stn["M"]
    h = x1n.T @ x1                    # = G + Gamma
    d = x1n - x1
    n2_x1 = np.sum(d * d)             # = tr(Omega)
    x2sq = np.sum(m * c) + np.sum(st["lam"])
    x2nsq = np.sum(mn * cn) + np.sum(stn["lam"])
    # cross term, expanded so that only k x k, k x b, b x b products appear
    cv, cnvn = c @ v, cn @ vn                                   # k x b, k x b'
    hc = h @ c                                                  # k x (n-k)
    t1 = (np.sum(cn * hc) - np.sum((cn @ v) * (h @ cv)) - np.sum(cnvn * (hc @ vn))
          + np.sum((vn.T @ v) * (cnvn.T @ h @ cv)))
    t2 = np.sum((mn @ v) * (cn @ v)) - np.sum((vn.T @ v) * (cnvn.T @ (mn @ v)))
    t3 = np.sum((m @ vn) * (c @ vn)) - np.sum((v.T @ vn) * (cv.T @ (m @ vn)))
    t4 = np.sum((vn.T @ ga @ v) * (vn.T @ v))
    cross = t1 + t2 + t3 + t4
    return n2_x1 + x2nsq + x2sq - 2.0 * cross
