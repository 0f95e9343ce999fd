"""Field evaluation, Mie series, incident fields and the superellipsoid
generator on the CPU: the oracle's layer sums and the host Mie/dipole
restatements are pinned to fixtures made by the unmodified reference
(tests/golden/fields.npz); the reference's own analytic tests
(test_reference.py:33-146) are restated."""

import numpy as np
import pytest

import oracle
from _support import GOLDEN, rel
from paper_2408_02274_b200 import surface
from paper_2408_02274_b200.fields import (electric_dipole, fibonacci_sphere,
                                          gaussian_beam, mie_solution,
                                          plane_wave)
from paper_2408_02274_b200.operator import MaterialPair

OMEGA = 2 * np.pi
Z = dict(np.load(GOLDEN / "fields.npz"))


def fd_curl(field, x, h=1e-5):
    c = np.zeros(3, dtype=complex)
    for i, j, k in ((0, 1, 2), (1, 2, 0), (2, 0, 1)):
        for a, b, sg in ((j, k, 1.0), (k, j, -1.0)):
            xp, xm = x.copy(), x.copy()
            xp[a] += h
            xm[a] -= h
            c[i] += sg * (field(xp)[b] - field(xm)[b]) / (2 * h)
    return c


def test_oracle_layer_fields_vs_reference_golden():
    disc = surface.make_sphere_surface(1, 10)
    mats = MaterialPair(1.0, 1.0, 2.25, 1.0, OMEGA)
    for pts, kap, key in ((Z["p_in"], mats.kappa_i, "lf_in"),
                          (Z["p_out"], mats.kappa_e, "lf_out")):
        got = oracle.layer_fields(pts, disc.points, disc.weights, Z["s1_m"],
                                  Z["s1_j"], kap)
        assert rel(got, Z[key]) < 1e-13


def test_mie_coefficients_and_fields_vs_reference_golden():
    mats = MaterialPair(1.0, 1.0, 2.25, 1.0, OMEGA)
    mie = mie_solution(1.0, mats)
    for k in "abcd":
        assert rel(getattr(mie, k), Z[f"mie_{k}"]) < 1e-13
    e, h = mie.interior_fields(Z["pm_in"])
    assert rel(e, Z["mie_e_in"]) < 1e-12 and rel(h, Z["mie_h_in"]) < 1e-12
    e, h = mie.exterior_scattered(Z["pm_out"])
    assert rel(e, Z["mie_e_sc"]) < 1e-12 and rel(h, Z["mie_h_sc"]) < 1e-12


def test_dipole_vs_reference_golden():
    dip = electric_dipole([0.1, -0.2, 0.3], [1.0, 0.5j, -0.25], eps=2.0,
                          omega=OMEGA)
    e, h = dip.fields(Z["pm_out"])
    assert rel(e, Z["dip_e"]) < 1e-13 and rel(h, Z["dip_h"]) < 1e-13


def test_mie_matched_media_no_scattering():
    mats = MaterialPair(1.0, 1.0, 1.0, 1.0, OMEGA)
    mie = mie_solution(1.0, mats)
    assert np.abs(mie.a).max() == 0.0 and np.abs(mie.b).max() == 0.0
    pts = fibonacci_sphere(40, 0.6)
    e, h = mie.interior_fields(pts)
    ei, hi = plane_wave(mats.kappa_e, omega=OMEGA).fields(pts)
    assert np.abs(e - ei).max() < 1e-10 and np.abs(h - hi).max() < 1e-10


def test_mie_transmission_conditions():
    mats = MaterialPair(1.0, 1.0, 2.25, 1.0, OMEGA)
    mie = mie_solution(1.0, mats)
    pts = fibonacci_sphere(100, 1.0)
    ei, hi = mie.interior_fields(pts)
    ee, he = mie.exterior_total(pts)
    for a, b in ((ei, ee), (hi, he)):
        scale = np.abs(np.cross(pts, b)).max()
        assert np.abs(np.cross(pts, a) - np.cross(pts, b)).max() < 1e-8 * scale


def test_mie_maxwell_and_guards():
    mats = MaterialPair(1.0, 1.0, 2.25, 1.0, OMEGA)
    mie = mie_solution(1.0, mats)
    fe = lambda x: mie.interior_fields(x[None])[0][0]
    fh = lambda x: mie.interior_fields(x[None])[1][0]
    x = np.array([0.1, -0.2, 0.15])
    scale = np.abs(fh(x)).max() + 1.0
    assert np.abs(fd_curl(fe, x) - 1j * OMEGA * mats.mu_i * fh(x)).max() < 1e-5 * scale
    with pytest.raises(ValueError):
        mie.interior_fields([[0.0, 0.0, 2.0]])
    with pytest.raises(ValueError):
        mie.exterior_scattered([[0.0, 0.0, 0.5]])


@pytest.mark.parametrize("make", [
    lambda: plane_wave(OMEGA, omega=OMEGA),
    lambda: electric_dipole([0.0, 0.1, -0.2], [0.3, 1.0, 0.2j], omega=OMEGA),
    lambda: gaussian_beam(OMEGA, focus=(0.0, 0.0, -3.0), waist=1.2, omega=OMEGA),
])
def test_incident_fields_satisfy_maxwell(make):
    inc = make()
    fe = lambda x: inc.fields(x[None])[0][0]
    fh = lambda x: inc.fields(x[None])[1][0]
    rng = np.random.default_rng(0)
    for _ in range(3):
        x = rng.normal(size=3) * 0.5
        s = np.abs(fe(x)).max() + np.abs(fh(x)).max()
        assert np.abs(fd_curl(fe, x) - 1j * OMEGA * fh(x)).max() < 1e-6 * s
        assert np.abs(fd_curl(fh, x) + 1j * OMEGA * fe(x)).max() < 1e-6 * s


def test_gaussian_beam_profile():
    k = 2 * np.pi
    gb = gaussian_beam(k, focus=(0.0, 0.0, 0.0), waist=1.5, omega=k)
    e0 = gb.fields([[0.0, 0.0, 1.5e-6]])[0][0]
    assert abs(np.linalg.norm(e0) - 1.0) < 1e-12
    # Gaussian transverse profile near the waist: |E(w0)| ~ exp(-1) |E(0)|
    ez = gb.fields([[0.0, 0.0, 0.01]])[0][0]
    ew = gb.fields([[1.5, 0.0, 0.01]])[0][0]
    assert abs(np.linalg.norm(ew) / np.linalg.norm(ez) - np.exp(-1.0)) < 0.03
    # propagates along +z: phase advances as exp(i k z) near the axis
    e1 = gb.fields([[0.0, 0.0, 0.06]])[0][0][0]
    assert abs(np.angle(e1 / ez[0]) - k * 0.05) < 0.02
    # upstream of the waist plane the field is exponentially small
    assert np.linalg.norm(gb.fields([[0.0, 0.0, -0.5]])[0][0]) < 1e-6
    with pytest.raises(ValueError):
        gaussian_beam(k, polarization=(0.0, 0.0, 1.0))


def test_superellipsoid_surface():
    a = (2.0, 1.0, 0.5)
    d = surface.make_superellipsoid_surface(2, 8, a, 4.0)
    x = d.points
    resid = ((np.abs(x / a) ** 4).sum(1) - 1.0)
    assert np.abs(resid).max() < 1e-8
    assert np.all(np.einsum("ij,ij->i", d.normals, x) > 0)
    assert d.n_patches == 6 * 4 and d.n_points == 24 * 64
    # exponent 2, unit axes: the sphere (area 4 pi)
    s = surface.make_superellipsoid_surface(2, 10, (1, 1, 1), 2.0)
    assert abs(s.area() - 4 * np.pi) < 1e-6
    # aspect-graded splits (n_x, n_y, n_z): faces normal to x get n_y * n_z
    g = surface.make_superellipsoid_surface((4, 2, 1), 6, (8, 1, 0.5), 8.0)
    assert g.n_patches == 2 * (2 * 1 + 4 * 1 + 4 * 2)
    with pytest.raises(ValueError):
        surface.make_superellipsoid_surface(0, 6)
