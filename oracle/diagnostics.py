"""Error metrics and the paper's propositions as executable checks.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np


def fro(a) -> float:
    return float(np.linalg.norm(np.asarray(a, dtype=np.float64)))


def quant_error(x, w, qx, qw) -> float:
    """E(X, W) = ||XW - Q(X)Q(W)||_F  (Eq. 3)."""
    x = np.asarray(x, np.float64)
    w = np.asarray(w, np.float64)
    return fro(x @ w - np.asarray(qx, np.float64) @ np.asarray(qw, np.float64))


def prop41_bound(x, w, qx, qw) -> float:
    """Right side of Prop. 4.1:
    ||X|| ||W - Q(W)|| + ||X - Q(X)|| (||W|| + ||W - Q(W)||)."""
    ew = fro(np.asarray(w, np.float64) - qw)
    ex = fro(np.asarray(x, np.float64) - qx)
    return fro(x) * ew + ex * (fro(w) + ew)


def prop42_gaussian_c(size: int) -> float:
    """c = sqrt(log(size) pi / size) for Gaussian R (natural log)."""
    return float(np.sqrt(np.log(size) * np.pi / size))


def prop42_rhs(size: int, q_max: float, mean_fro_r: float) -> float:
    """c sqrt(size) / q_max * E||R||_F  (Prop. 4.2)."""
    return prop42_gaussian_c(size) * np.sqrt(size) / q_max * mean_fro_r


def lowrank_cost_fraction(m: int, n: int, r: int) -> float:
    """Extra parameters / compute of the low-rank branch: (mr + nr) / (mn)."""
    return (m * r + n * r) / (m * n)


def residual_norm_closed_form(sigma, r: int) -> float:
    """||R||_F = sqrt(sum_{i > r} sigma_i^2)."""
    s = np.asarray(sigma, np.float64)
    return float(np.sqrt(np.sum(s[r:] ** 2)))


def rel_fro(a, b) -> float:
    """||a - b||_F / ||b||_F."""
    b = np.asarray(b, np.float64)
    d = np.asarray(a, np.float64) - b
    nb = fro(b)
    return fro(d) / nb if nb else fro(d)
