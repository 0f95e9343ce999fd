"""Open (first-kind) Chebyshev grid primitives used at plan time.

Host-side plan inputs only (no device work here).  Every routine evaluates the
same floating-point expression, in the same order, as the reference so the
plan integers built on top of it (segment ids, singular classification) come
out bit-identical on the same host:

* nodes            -- reference ``chebyshev.py:60-65``  (cos((k+1/2)pi/n), decreasing)
* fejer weights    -- reference ``chebyshev.py:68-79``
* basis recurrence -- reference ``chebyshev.py:82-95``  (legal slightly outside [-1,1])
* values->coeffs   -- reference ``chebyshev.py:98-105``
* derivative       -- reference ``chebyshev.py:113-138``
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

__all__ = ["nodes", "fejer", "basis", "to_coeff_matrix", "deriv_series",
           "diff_matrix", "eval_matrix"]


@lru_cache(maxsize=64)
def _nodes_cached(n: int) -> np.ndarray:
    k = np.arange(n)
    out = np.cos((k + 0.5) * np.pi / n)
    out.setflags(write=False)
    return out


def nodes(n: int) -> np.ndarray:
    """n open Chebyshev nodes, listed with decreasing value."""
    if n < 1:
        raise ValueError("node count must be positive")
    return _nodes_cached(n)


def fejer(n: int) -> np.ndarray:
    """Fejer first-rule weights on ``nodes(n)`` (sum to 2)."""
    if n < 1:
        raise ValueError("node count must be positive")
    ang = (np.arange(n) + 0.5) * np.pi / n
    m = np.arange(1, n // 2 + 1)
    if m.size == 0:
        return np.full(n, 2.0 / n)
    terms = np.cos(2.0 * np.outer(ang, m)) / (4.0 * m**2 - 1.0)
    return (2.0 / n) * (1.0 - 2.0 * terms.sum(axis=1))


def basis(n: int, x) -> np.ndarray:
    """T_0..T_{n-1} at x via the three-term recurrence, shape (len(x), n)."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    tab = np.empty((x.size, n))
    tab[:, 0] = 1.0
    if n > 1:
        tab[:, 1] = x
    for i in range(2, n):
        tab[:, i] = 2.0 * x * tab[:, i - 1] - tab[:, i - 2]
    return tab


@lru_cache(maxsize=64)
def to_coeff_matrix(n: int) -> np.ndarray:
    """Samples on ``nodes(n)`` -> Chebyshev series coefficients."""
    mat = (2.0 / n) * basis(n, nodes(n)).T
    mat[0] *= 0.5
    mat.setflags(write=False)
    return mat


@lru_cache(maxsize=64)
def eval_matrix(n: int) -> np.ndarray:
    out = basis(n, nodes(n))
    out.setflags(write=False)
    return out


def deriv_series(coeffs: np.ndarray) -> np.ndarray:
    """Series coefficients of the derivative (backward recurrence)."""
    n = coeffs.shape[0]
    res = np.zeros_like(coeffs)
    if n < 2:
        return res
    for k in range(n - 1, 0, -1):
        nxt = res[k + 1] if k + 1 < n else 0.0
        res[k - 1] = nxt + 2.0 * k * coeffs[k]
    res[0] *= 0.5
    return res


@lru_cache(maxsize=64)
def diff_matrix(n: int) -> np.ndarray:
    """Spectral differentiation on the n-point open grid (samples -> samples)."""
    if n < 2:
        raise ValueError("need at least two nodes to differentiate")
    dcoef = np.zeros((n, n))
    for col in range(n):
        unit = np.zeros(n)
        unit[col] = 1.0
        dcoef[:, col] = deriv_series(unit)
    out = eval_matrix(n) @ dcoef @ to_coeff_matrix(n)
    out.setflags(write=False)
    return out
