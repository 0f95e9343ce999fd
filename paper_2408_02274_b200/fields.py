"""Incident fields used to form GMRES right-hand sides (host, plan time).

``plane_wave`` restates reference ``reference.py:41-64``
(E = pol exp(i kappa d.x), H = kappa/(omega mu) (d x pol) exp(i kappa d.x)).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["IncidentField", "plane_wave"]


@dataclass
class IncidentField:
    kind: str
    fields: callable
    kappa: complex


def plane_wave(kappa_e, direction=(0.0, 0.0, -1.0),
               polarization=(1.0, 0.0, 0.0), omega=None,
               mu_e=1.0) -> IncidentField:
    d = np.asarray(direction, dtype=float)
    p = np.asarray(polarization, dtype=complex)
    if abs(np.linalg.norm(d) - 1.0) > 1e-12:
        raise ValueError("direction must be a unit vector")
    if abs(np.vdot(d, p)) > 1e-12:
        raise ValueError("polarization must be orthogonal to direction")
    omega = float(omega if omega is not None else np.real(kappa_e))
    h_pol = kappa_e / (omega * mu_e) * np.cross(d, p)

    def fields(points):
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        phase = np.exp(1j * kappa_e * (pts @ d))
        return np.outer(phase, p), np.outer(phase, h_pol)

    return IncidentField("plane-wave", fields, kappa_e)
