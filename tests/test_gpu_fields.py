"""GPU off-surface field evaluation (ifgfb_layer_fields, csrc/fields.cu)
against the unmodified reference's fixtures (tests/golden/fields.npz) and
the oracle, the reference's evaluate_fields tests restated
(test_reference.py:150-230), and the validate-sphere loop (cli.py:258-289):
cfg-1 GMRES on the device, interior fields vs the Mie series.

Tolerances: the layer sums are an O(N) direct reduction in FP64 whose
summation order differs from numpy's: 1e-12 relative l2."""

import numpy as np
import pytest

import oracle
from _support import GOLDEN, inputs, plan_matches_golden, rel
from paper_2408_02274_b200 import surface
from paper_2408_02274_b200.fields import (evaluate_fields, fibonacci_sphere,
                                          layer_fields, mie_solution,
                                          plane_wave)
from paper_2408_02274_b200.operator import (DensityBlock, MaterialPair,
                                            MullerOperator)
from paper_2408_02274_b200.solver import gmres

pytestmark = pytest.mark.gpu

OMEGA = 2 * np.pi
Z = dict(np.load(GOLDEN / "fields.npz"))
MATS = MaterialPair(1.0, 1.0, 2.25, 1.0, OMEGA)


def s1_density():
    disc = surface.make_sphere_surface(1, 10)
    return disc, DensityBlock.from_currents(disc, Z["s1_j"], Z["s1_m"])


def test_layer_fields_vs_reference_golden_and_oracle():
    disc, dens = s1_density()
    for pts, kap, key in ((Z["p_in"], MATS.kappa_i, "lf_in"),
                          (Z["p_out"], MATS.kappa_e, "lf_out")):
        got, dmin = layer_fields(disc, dens, kap, pts)
        assert rel(got, Z[key]) < 1e-12
        ref = oracle.layer_fields(pts, disc.points, disc.weights, dens.m, dens.j, kap)
        assert rel(got, ref) < 1e-12
        d_ref = np.min(np.linalg.norm(pts[:, None] - disc.points[None], axis=-1), 1)
        assert np.array_equal(dmin, d_ref) or np.abs(dmin - d_ref).max() < 1e-15
    # deterministic: bitwise run to run
    a, _ = layer_fields(disc, dens, MATS.kappa_i, Z["p_in"])
    b, _ = layer_fields(disc, dens, MATS.kappa_i, Z["p_in"])
    assert np.array_equal(a, b)


def test_layer_fields_complex_wavenumber_vs_oracle():
    disc, dens = s1_density()
    kap = 2 * np.pi * (1.2 + 0.3j)     # lossy medium
    got, _ = layer_fields(disc, dens, kap, Z["p_in"])
    ref = oracle.layer_fields(Z["p_in"], disc.points, disc.weights, dens.m, dens.j, kap)
    assert rel(got, ref) < 1e-12


def test_evaluate_fields_vs_reference_golden():
    disc, dens = s1_density()
    e, h = evaluate_fields(disc, dens, MATS, Z["p_in"], "interior")
    assert rel(e, Z["e_in"]) < 1e-12 and rel(h, Z["h_in"]) < 1e-12
    inc = plane_wave(OMEGA, omega=OMEGA)
    e, h = evaluate_fields(disc, dens, MATS, Z["p_out"], "exterior", incident=inc)
    assert rel(e, Z["e_out"]) < 1e-12 and rel(h, Z["h_out"]) < 1e-12


def test_evaluate_fields_zero_density_and_guards():
    disc = surface.make_sphere_surface(1, 10)
    dens = DensityBlock(np.zeros((8, disc.n_points), dtype=complex))
    pw = plane_wave(MATS.kappa_e, omega=OMEGA)
    pts = np.array([[0.0, 0.0, 3.0]])
    e, h = evaluate_fields(disc, dens, MATS, pts, "exterior", incident=pw)
    e_ref, _ = pw.fields(pts)
    assert np.abs(e - e_ref).max() < 1e-14
    e0, _ = evaluate_fields(disc, dens, MATS, pts, "exterior")
    assert np.abs(e0).max() == 0.0
    with pytest.raises(ValueError):
        evaluate_fields(disc, dens, MATS, disc.points[:1] * 1.0001, "exterior")
    with pytest.raises(ValueError):
        evaluate_fields(disc, dens, MATS, pts, "sideways")
    out, _ = layer_fields(disc, dens, MATS.kappa_e, np.zeros((0, 3)))
    assert out.shape == (4, 0, 3)


def test_extinction_identity():
    """Matched media: currents of an interior Maxwell field reproduce it
    inside and cancel outside (reference test_reference.py:150-170)."""
    mats = MaterialPair(1.0, 1.0, 1.0, 1.0, OMEGA)
    disc = surface.make_sphere_surface(2, 12)
    pw = plane_wave(mats.kappa_e, omega=OMEGA)
    e, h = pw.fields(disc.points)
    n = disc.normals
    dens = DensityBlock.from_currents(disc, np.cross(n, h) / OMEGA,
                                      np.cross(n, e) / OMEGA)
    pin = np.array([[0.2, -0.1, 0.3], [0.0, 0.0, 0.0]])
    e_in, h_in = evaluate_fields(disc, dens, mats, pin, "interior")
    e_ref, h_ref = pw.fields(pin)
    assert np.abs(e_in - e_ref).max() < 1e-5 and np.abs(h_in - h_ref).max() < 1e-5
    pout = np.array([[2.0, 0.5, -0.3], [0.0, -2.5, 1.0]])
    e_out, h_out = evaluate_fields(disc, dens, mats, pout, "exterior")
    assert np.abs(e_out).max() < 1e-5 and np.abs(h_out).max() < 1e-5


def test_validate_sphere_cfg1_against_mie():
    """cfg 1 GMRES on the device, then the interior field at 1,000 points
    against the series solution (the reference's validate-sphere check).
    The reference's own error on its own solution is in the fixture."""
    if not plan_matches_golden("c1"):
        pytest.skip("host numpy produced a different plan than the golden host")
    inp = inputs("c1")
    op = MullerOperator(inp["disc"], inp["mats"], inp["smap"], inp["moments"],
                        (inp["corr"].ell_idx, inp["corr"].src_idx),
                        tree=inp["tree"], hierarchy=inp["hier"])
    b = op.rhs(plane_wave(OMEGA, direction=(0.0, 0.0, 1.0), omega=OMEGA))
    x, rep = gmres(op, b, tol=1e-6, max_iter=300)
    assert rep.converged
    m, j = op.decode(x)
    dens = DensityBlock.from_currents(op.disc, j, m)
    pv = fibonacci_sphere(1000, 0.7)
    e, h = evaluate_fields(op.disc, dens, op.materials, pv, "interior")
    assert rel(e, Z["val_e"]) < 1e-7 and rel(h, Z["val_h"]) < 1e-7
    e_ref, h_ref = mie_solution(1.0, op.materials)._eval(pv, "interior")
    err_e, err_h = rel(e, e_ref), rel(h, h_ref)
    assert abs(err_e - float(Z["val_err_e"])) < 1e-8
    assert abs(err_h - float(Z["val_err_h"])) < 1e-8
    assert err_e < 1e-2 and err_h < 1e-2
