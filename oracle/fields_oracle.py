"""CPU ORACLE (test infrastructure only -- never imported by the product).

numpy restatement of the off-surface layer sums of reference
reference.py:285-312 (_layer_fields): curl S[m], curl S[j], curlcurl S[m],
curlcurl S[j] at targets from weighted surface currents, kernel
G = exp(i kappa r)/(4 pi r).  Pinned against tests/golden/fields.npz
(tests/test_fields.py).
"""

from __future__ import annotations

import numpy as np


def layer_fields(points, src_points, weights, m, j, kappa, block=1024):
    """(4, M, 3) complex, rows in the reference's order (reference.py:291)."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    mw = np.asarray(m) * weights[:, None]
    jw = np.asarray(j) * weights[:, None]
    out = np.zeros((4, pts.shape[0], 3), dtype=complex)
    for t0 in range(0, pts.shape[0], block):
        t1 = min(t0 + block, pts.shape[0])
        dx = pts[t0:t1, None, :] - src_points[None, :, :]       # (t, s, 3)
        r2 = (dx * dx).sum(-1)
        r = np.sqrt(r2)
        g = np.exp(1j * kappa * r) / (4.0 * np.pi * r)
        a = (1j * kappa * r - 1.0) / r2                          # grad G = G a dx
        bb = (3.0 - 3.0 * (1j * kappa * r) - kappa**2 * r2) / r2
        for row, w in ((0, mw), (1, jw)):
            out[row, t0:t1] = np.cross((g * a)[:, :, None] * dx,
                                       np.broadcast_to(w, dx.shape)).sum(1)
        for row, w in ((2, mw), (3, jw)):
            proj = np.einsum("tsc,sc->ts", dx, w) / r2
            out[row, t0:t1] = ((g * (a + kappa**2))[:, :, None] * w[None] +
                               (g * bb * proj)[:, :, None] * dx).sum(1)
    return out
