"""CPU emulation of one device system solve, for host-side pattern tests.

Evaluates a `discretization.Pattern` for a K field into a dense matrix
(interior band + border), solves it with numpy, and applies the same
readouts as the device `extract` kernel. Test helper only.
"""

import numpy as np


def term_values(kind, c, k, K):
    K = np.asarray(K, dtype=float)
    kk = K[k] if len(K) else np.ones(len(k))
    return np.where(kind == 1, c / kk, np.where(kind == 2, c / np.sqrt(kk), c))


def dense_system(pat, K):
    """Interior matrix K_II (n x n) and the rhs block over rows I and J."""
    n, nb = pat.n, pat.nb
    A = np.zeros((n, n))
    vals = np.add.reduceat(term_values(pat.t_kind, pat.t_c, pat.t_k, K), pat.e_tptr[:-1]) \
        if len(pat.e_row) else np.zeros(0)
    A[pat.e_row, pat.e_col] = vals
    rhs = np.zeros((n + nb, pat.ndof + 1))
    for d in range(pat.ndof):
        sl = slice(pat.q_ptr[d], pat.q_ptr[d + 1])
        rhs[pat.q_row[sl], d] = pat.q_val[sl]
    rhs[:, pat.ndof] = pat.bar_const
    if len(pat.b_row):
        bv = np.add.reduceat(term_values(pat.bt_kind, pat.bt_c, pat.bt_k, K), pat.b_tptr[:-1])
        rhs[pat.b_row, pat.ndof] += bv
    return A, rhs


def solve(pat, K):
    """Mirror of band_solve_kernel: compatible rhs, pinned solve, projection."""
    A, rhs = dense_system(pat, K)
    n, nb = pat.n, pat.nb
    if nb:
        Cf = np.zeros((nb, n + nb))
        Cf[:, :n] = pat.E.T
        Cf[:, n:] = pat.G[:nb]
        Ci = pat.G[nb:]
        mu = Ci @ (Cf @ rhs)
        rt = rhs - Cf.T @ mu
        Xt = np.zeros_like(rhs)
        Xt[:n] = np.linalg.solve(A, rt[:n])
        X = Xt - Cf.T @ (Ci @ (Cf @ Xt))
    else:
        X = np.linalg.solve(A, rhs)
    nd = pat.ndof
    Q = np.zeros((pat.n + pat.nb, nd))
    for d in range(nd):
        sl = slice(pat.q_ptr[d], pat.q_ptr[d + 1])
        Q[pat.q_row[sl], d] = pat.q_val[sl]
    B = Q.T @ X[:, :nd]
    h = Q.T @ X[:, nd] + pat.h_lift
    P = np.zeros((pat.nfield, pat.n + pat.nb))
    for f in range(pat.nfield):
        sl = slice(pat.p_ptr[f], pat.p_ptr[f + 1])
        P[f, pat.p_col[sl]] += pat.p_val[sl]
    M = P @ X[:, :nd]
    Fb = P @ X[:, nd] + pat.f_lift
    return {"B": B, "h": h, "M": M, "Fb": Fb, "X": X, "A": A}
