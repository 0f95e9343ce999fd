"""Incident fields, the dielectric-sphere series solution and off-surface
field evaluation (closes the validate-sphere loop).

* ``plane_wave`` restates reference ``reference.py:41-64``
  (E = pol exp(i kappa d.x), H = kappa/(omega mu) (d x pol) exp(i kappa d.x)).
* ``electric_dipole`` restates ``reference.py:67-95``; ``gaussian_beam``
  (not in the reference; BASELINE config 4 asks for it) is the
  complex-source-point beam, i.e. the same dipole placed at the complex
  position focus + i b d, an exact Maxwell solution whose waist is
  w0 = sqrt(2 b / kappa).
* ``mie_solution`` / ``MieSolution`` restate the classical series of
  ``reference.py:98-269`` (host, scipy Bessel functions, validation only).
* ``evaluate_fields`` mirrors ``reference.py:315-347``; its O(M N) layer
  sums (``_layer_fields``, ``reference.py:285-312``) run on the GPU through
  ``ifgfb_layer_fields`` (csrc/fields.cu).  There is no CPU fallback.

Conventions (reference.py:1-8): time dependence exp(-i omega t), curl E =
i omega mu H, curl H = -i omega eps E, kernel exp(i kappa r)/(4 pi r).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["IncidentField", "MieSolution", "plane_wave", "electric_dipole",
           "gaussian_beam", "mie_solution", "evaluate_fields",
           "layer_fields", "fibonacci_sphere"]


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


def _dipole_fields(pts, y0, p, kappa, omega, mu):
    """Dipole fields with a (possibly complex) source position y0:
    E = i omega mu (G p + grad div (G p) / kappa^2), H = grad G x p, with
    grad grad G = G (a I + b rhat rhat), a = (i kappa r - 1)/r^2,
    b = (3 - 3 i kappa r - kappa^2 r^2)/r^2 (reference.py:67-95).  For a
    complex y0, r is the principal square root of (x - y0).(x - y0)."""
    dx = pts.astype(complex) - y0
    r = np.sqrt((dx * dx).sum(axis=1))
    if np.any(r == 0.0):
        raise ValueError("evaluation at the dipole position")
    rhat = dx / r[:, None]
    g = np.exp(1j * kappa * r) / (4.0 * np.pi * r)
    ikr = 1j * kappa * r
    a = (ikr - 1.0) / r**2
    b = (3.0 - 3.0 * ikr - kappa**2 * r**2) / r**2
    rp = rhat @ p
    e = 1j * omega * mu * ((g * (1.0 + a / kappa**2))[:, None] * p[None, :]
                           + (g * b * rp / kappa**2)[:, None] * rhat)
    h = np.cross((g * a * r)[:, None] * rhat, np.broadcast_to(p, rhat.shape))
    return e, h


def electric_dipole(position, moment, eps=1.0, mu=1.0, omega=1.0) -> IncidentField:
    y0 = np.asarray(position, dtype=float)
    p = np.asarray(moment, dtype=complex)
    kappa = omega * np.sqrt(eps * mu)

    def fields(points):
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        return _dipole_fields(pts, y0, p, kappa, omega, mu)

    return IncidentField("dipole", fields, kappa)


def gaussian_beam(kappa_e, focus=(0.0, 0.0, 0.0), direction=(0.0, 0.0, 1.0),
                  polarization=(1.0, 0.0, 0.0), waist=None, omega=None,
                  mu_e=1.0) -> IncidentField:
    """Complex-source-point Gaussian beam travelling along ``direction`` with
    its waist ``waist`` (default 2 wavelengths) in the plane through
    ``focus`` normal to the axis; |E| = 1 on the axis just downstream of the
    waist.  The dipole sits at focus + i b d with b = kappa w0^2 / 2; with
    the principal square root the field is an exact Maxwell solution off
    the branch disc (radius b in the waist plane), Gaussian downstream of it
    (|E| ~ exp(-rho^2 / w0^2) near the waist) and exponentially small
    (exp(-2 kappa b)) upstream: place the scatterer downstream of the waist
    plane."""
    d = np.asarray(direction, dtype=float)
    p = np.asarray(polarization, dtype=complex)
    if abs(np.linalg.norm(d) - 1.0) > 1e-12:
        raise ValueError("direction must be a unit vector")
    if abs(np.vdot(d, p)) > 1e-12:
        raise ValueError("polarization must be orthogonal to direction")
    omega = float(omega if omega is not None else np.real(kappa_e))
    kr = float(np.real(kappa_e))
    w0 = float(waist) if waist is not None else 2.0 * (2.0 * np.pi / kr)
    if not w0 > 0:
        raise ValueError("waist must be positive")
    b = 0.5 * kr * w0 * w0
    f = np.asarray(focus, dtype=float)
    y0 = f + 1j * b * d
    # on-axis reference point 1e-6 w0 downstream of the waist (the waist
    # plane itself is the branch disc)
    e_f, _ = _dipole_fields((f + 1e-6 * w0 * d)[None, :], y0, p, kappa_e, omega, mu_e)
    scale = 1.0 / np.linalg.norm(e_f[0])

    def fields(points):
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        e, h = _dipole_fields(pts, y0, p, kappa_e, omega, mu_e)
        return e * scale, h * scale

    return IncidentField("gaussian-beam", fields, kappa_e)


# ---------------------------------------------------------------------------
# dielectric sphere series (host; validation only)
# ---------------------------------------------------------------------------

def _sph_j(n, z, derivative=False):
    from scipy.special import spherical_jn
    return spherical_jn(n, np.real_if_close(z), derivative)


def _sph_h1(n, z, derivative=False):
    from scipy.special import spherical_jn, spherical_yn
    z = np.real_if_close(z)
    return spherical_jn(n, z, derivative) + 1j * spherical_yn(n, z, derivative)


def _pi_tau(n_max, mu):
    """Angular functions pi_n, tau_n (n = 1..n_max) at cos(theta) = mu."""
    pi = np.zeros((n_max + 1,) + mu.shape)
    pi[1] = 1.0
    for n in range(1, n_max):
        pi[n + 1] = ((2 * n + 1) * mu * pi[n] - (n + 1) * pi[n - 1]) / n
    n = np.arange(1, n_max + 1)[:, None]
    tau = n * mu * pi[1:] - (n + 1) * pi[:-1]
    return pi[1:], tau


@dataclass
class MieSolution:
    radius: float
    materials: object
    order: int
    a: np.ndarray
    b: np.ndarray
    c: np.ndarray
    d: np.ndarray

    def _eval(self, points, region):
        """Incidence exp(+i k z) x_hat: interior total or exterior
        scattered field (reference.py:136-213)."""
        mats = self.materials
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        r = np.linalg.norm(pts, axis=1)
        if region == "interior" and np.any(r > self.radius * (1 + 1e-12)):
            raise ValueError("interior evaluator used outside the sphere")
        if region == "exterior" and np.any(r < self.radius * (1 - 1e-12)):
            raise ValueError("exterior evaluator used inside the sphere")
        r = np.where(r == 0.0, 1e-300, r)
        ct = np.clip(pts[:, 2] / r, -1.0, 1.0)
        st = np.sqrt(np.maximum(0.0, 1.0 - ct * ct))
        ph = np.arctan2(pts[:, 1], pts[:, 0])
        cp, sp = np.cos(ph), np.sin(ph)
        nn = np.arange(1, self.order + 1)
        if region == "interior":
            kap, cm, cn, zf = mats.kappa_i, self.c, self.d, _sph_j
            ofac = mats.kappa_i / (mats.omega * mats.mu_i)
            sgn = 1.0
        else:
            kap, cm, cn, zf = mats.kappa_e, self.b, self.a, _sph_h1
            ofac = mats.kappa_e / (mats.omega * mats.mu_e)
            sgn = -1.0
        rho = kap * r
        z = np.stack([zf(n, rho) for n in nn])
        zeta = z / rho + np.stack([zf(n, rho, True) for n in nn])
        pi_n, tau_n = _pi_tau(self.order, ct)
        en = (1j ** nn * (2 * nn + 1) / (nn * (nn + 1.0)))[:, None]
        nn1 = (nn * (nn + 1.0))[:, None]

        def harmonics(fm, fn, even):
            # (M_o1n, N_e1n) for E (even = True), (M_e1n, N_o1n) for H
            c1, c2 = (cp, sp) if even else (sp, cp)
            sg = 1.0 if even else -1.0
            m_t = sg * c1 * pi_n * z
            m_p = -c2 * tau_n * z
            n_r = c1 * st * nn1 * pi_n * z / rho
            n_t = c1 * tau_n * zeta
            n_p = -sg * c2 * pi_n * zeta
            return ((en * fn * n_r).sum(0), (en * (fm * m_t + fn * n_t)).sum(0),
                    (en * (fm * m_p + fn * n_p)).sum(0))

        cm, cn = cm[:, None], cn[:, None]
        er, et, ep = harmonics(sgn * cm, -sgn * 1j * cn, True)
        hr, ht, hp = harmonics(-sgn * ofac * cn, -sgn * 1j * ofac * cm, False)
        rh = np.stack([st * cp, st * sp, ct], 1)
        th = np.stack([ct * cp, ct * sp, -st], 1)
        phh = np.stack([-sp, cp, np.zeros_like(sp)], 1)
        e = er[:, None] * rh + et[:, None] * th + ep[:, None] * phh
        h = hr[:, None] * rh + ht[:, None] * th + hp[:, None] * phh
        return e, h

    def _rotated(self, points, region):
        # the series assumes travel along +z; the incident wave travels along
        # -z: rotate by pi about x (reference.py:225-237)
        pts = np.atleast_2d(np.asarray(points, dtype=float)).copy()
        pts[:, 1:] *= -1.0
        e, h = self._eval(pts, region)
        e[:, 1:] *= -1.0
        h[:, 1:] *= -1.0
        return e, h

    def interior_fields(self, points):
        return self._rotated(points, "interior")

    def exterior_scattered(self, points):
        return self._rotated(points, "exterior")

    def exterior_total(self, points):
        e, h = self._rotated(points, "exterior")
        ei, hi = plane_wave(self.materials.kappa_e, omega=self.materials.omega,
                            mu_e=self.materials.mu_e).fields(points)
        return e + ei, h + hi


def mie_solution(radius: float, materials, order: int | None = None) -> MieSolution:
    """Series coefficients, truncation ceil(x + 8 x^(1/3) + 10) unless given
    (reference.py:240-269)."""
    x = materials.kappa_e * radius
    y = materials.kappa_i * radius
    if order is None:
        xa = abs(x)
        order = int(np.ceil(xa + 8.0 * xa ** (1.0 / 3.0) + 10.0))
    n = np.arange(1, order + 1)
    jx, jy, hx = _sph_j(n, x), _sph_j(n, y), _sph_h1(n, x)
    dpx = jx + x * _sph_j(n, x, True)       # [rho j_n]' at x
    dpy = jy + y * _sph_j(n, y, True)
    dxi = hx + x * _sph_h1(n, x, True)      # [rho h_n]' at x
    mu_e, mu_i = materials.mu_e, materials.mu_i
    mr = materials.kappa_i / materials.kappa_e
    b = (mu_i * dpx * jy - mu_e * jx * dpy) / (mu_i * dxi * jy - mu_e * hx * dpy)
    a = ((mu_i * dpy * jx - mr * mr * mu_e * jy * dpx) /
         (mu_i * dpy * hx - mr * mr * mu_e * jy * dxi))
    c = (jx - b * hx) / jy
    d = (mu_i / (mr * mu_e)) * (jx - a * hx) / jy
    return MieSolution(radius, materials, order, a, b, c, d)


def fibonacci_sphere(n: int, radius: float = 1.0) -> np.ndarray:
    """Golden-angle spiral points (reference.py:272-279)."""
    i = np.arange(n) + 0.5
    z = 1.0 - 2.0 * i / n
    phi = np.pi * (1.0 + np.sqrt(5.0)) * i
    st = np.sqrt(1.0 - z * z)
    return radius * np.stack([st * np.cos(phi), st * np.sin(phi), z], axis=1)


# ---------------------------------------------------------------------------
# off-surface fields (GPU)
# ---------------------------------------------------------------------------

def layer_fields(disc, dens, kappa, points):
    """(4, M, 3) complex: curl S[m], curl S[j], curlcurl S[m], curlcurl S[j]
    at ``points`` (reference _layer_fields, reference.py:285-312), and the
    (M,) minimum source distance; computed by ``ifgfb_layer_fields``."""
    lib = _lib.load()
    pts = np.ascontiguousarray(np.atleast_2d(np.asarray(points, dtype=float)))
    if pts.shape[1] != 3:
        raise ValueError("points must be (M, 3)")
    w = disc.weights[:, None]
    src = np.empty((disc.n_points, 15))
    src[:, 0:3] = disc.points
    src[:, 3:9] = np.ascontiguousarray(np.asarray(dens.m) * w).view(np.float64)
    src[:, 9:15] = np.ascontiguousarray(np.asarray(dens.j) * w).view(np.float64)
    out = np.empty((4, pts.shape[0], 3), dtype=complex)
    dmin = np.empty(pts.shape[0])
    kap = np.array([complex(kappa).real, complex(kappa).imag])
    _lib.check(lib.ifgfb_layer_fields(src.shape[0], _lib.dptr(src), pts.shape[0],
                                      _lib.dptr(pts), _lib.dptr(kap), _lib.dptr(out),
                                      _lib.dptr(dmin)), "layer_fields")
    return out, dmin


def evaluate_fields(disc, dens, materials, points, region: str,
                    incident: IncidentField | None = None,
                    min_distance: float | None = None):
    """(E, H) at off-surface points from surface currents (reference
    reference.py:315-347): E = -omega mu curl S[m] - i curlcurl S[j],
    H = -omega eps curl S[j] + i curlcurl S[m] with the region's wavenumber;
    interior = total field, exterior = scattered (+ incident if given).
    Points closer to the surface than ``min_distance`` (default: the largest
    classification radius) raise ValueError."""
    if region == "interior":
        kappa, eps, mu = materials.kappa_i, materials.eps_i, materials.mu_i
    elif region == "exterior":
        kappa, eps, mu = materials.kappa_e, materials.eps_e, materials.mu_e
    else:
        raise ValueError("region must be 'interior' or 'exterior'")
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    if min_distance is None:
        min_distance = float(disc.max_spacing.max())
    (curl_m, curl_j, cc_m, cc_j), dmin = layer_fields(disc, dens, kappa, pts)
    if np.any(dmin < min_distance):
        raise ValueError("evaluation points too close to the surface")
    omega = materials.omega
    e = -omega * mu * curl_m - 1j * cc_j
    h = -omega * eps * curl_j + 1j * cc_m
    if region == "exterior" and incident is not None:
        ei, hi = incident.fields(pts)
        e = e + ei
        h = h + hi
    return e, h
