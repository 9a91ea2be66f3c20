"""One-sided Jacobi SVD for tiny shapes, independent of LAPACK.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Used to pin the truncated-SVD step of SVDQuant ("the optimal solution
is L1 = U Sigma_{:, :r} and L2 = V_{:r, :}") on small matrices without
relying on the same LAPACK routine the default path calls.
"""
from __future__ import annotations

import numpy as np


def jacobi_svd(a, tol: float = 1e-15, max_sweeps: int = 100):
    """Return (U, s, Vt) with a = U diag(s) Vt, s descending, thin shapes.

    One-sided (Hestenes) Jacobi: orthogonalise the columns of a copy of `a`
    by plane rotations; column norms are the singular values.
    """
    a = np.array(a, dtype=np.float64)
    transpose = a.shape[0] < a.shape[1]
    if transpose:
        a = a.T
    m, n = a.shape
    U = a.copy()
    V = np.eye(n)
    for _ in range(max_sweeps):
        off = 0.0
        for p in range(n - 1):
            for q in range(p + 1, n):
                alpha = U[:, p] @ U[:, p]
                beta = U[:, q] @ U[:, q]
                gamma = U[:, p] @ U[:, q]
                if alpha == 0.0 or beta == 0.0:
                    continue
                c_off = abs(gamma) / np.sqrt(alpha * beta)
                off = max(off, c_off)
                if c_off < tol:
                    continue
                zeta = (beta - alpha) / (2.0 * gamma)
                t = np.sign(zeta) / (abs(zeta) + np.sqrt(1.0 + zeta * zeta)) if zeta != 0 else 1.0
                c = 1.0 / np.sqrt(1.0 + t * t)
                s = c * t
                up = U[:, p].copy()
                U[:, p] = c * up - s * U[:, q]
                U[:, q] = s * up + c * U[:, q]
                vp = V[:, p].copy()
                V[:, p] = c * vp - s * V[:, q]
                V[:, q] = s * vp + c * V[:, q]
        if off < tol:
            break
    sv = np.sqrt(np.sum(U * U, axis=0))
    order = np.argsort(-sv, kind="stable")
    sv = sv[order]
    U = U[:, order]
    V = V[:, order]
    nz = sv > 0
    U[:, nz] = U[:, nz] / sv[nz][None, :]
    if transpose:
        return V, sv, U.T
    return U, sv, V.T
