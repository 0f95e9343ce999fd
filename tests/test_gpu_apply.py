"""GPU N-Muller apply / potentials / GMRES against the unmodified reference
(golden), the oracle on this host, and the reference's operator and solver
tests (tests/test_operators.py, tests/test_solver.py) restated.

Tolerances (north star): apply(y) <= 1e-10 relative l2 (the reference's own
vec/seq floor is 2.8e-11 at cfg 1, 5.0e-11 at s1); raw far-field outputs <=
1e-13; GMRES residual history <= 1e-8 relative per entry.  D alone is NOT
held to 1e-10: the reference's own vec/seq runs differ by 2.2e-10 there
(finite difference with h = 1e-6)."""

import numpy as np
import pytest
import torch

import oracle
from _support import GOLDEN, golden, golden_rows, inputs, plan_matches_golden, rel
from paper_2408_02274_b200.fields import plane_wave
from paper_2408_02274_b200.operator import (DensityBlock, MullerOperator,
                                            build_muller_operator)
from paper_2408_02274_b200.solver import gmres

pytestmark = pytest.mark.gpu

_OPS = {}


def device_op(name) -> MullerOperator:
    if name not in _OPS:
        inp = inputs(name)
        _OPS[name] = MullerOperator(
            inp["disc"], inp["mats"], inp["smap"], inp["moments"],
            (inp["corr"].ell_idx, inp["corr"].src_idx), tree=inp["tree"],
            hierarchy=inp["hier"])
    return _OPS[name]


def _have(name):
    if not (GOLDEN / f"{name}.npz").exists():
        pytest.skip(f"{name} fixture not generated")


@pytest.mark.parametrize("name", ["s1", "c1", "se1", "sl1", "c2n4", "c2n8"])
def test_apply_vs_reference_golden(name):
    """c2n4 / c2n8: the benchmarked cfg-2 family at 38,400 and 153,600
    unknowns (sphere(4,10) k0 = 4 pi, sphere(8,10) k0 = 8 pi)."""
    _have(name)
    if not plan_matches_golden(name):
        pytest.skip("host numpy produced a different plan than the golden host")
    z = golden(name)
    op = device_op(name)
    out = op.apply(z["y"])
    # se1 (superellipsoid): the reference's own linearity floor is 1.5e-10
    # sl1 (short cfg-4 slab, eps_r 12.11): 3.6e-11
    assert rel(out, z["apply_y"]) < (1e-10 if name != "se1" else 3e-10)


@pytest.mark.parametrize("name", ["c1", "c2n4"])
def test_apply_with_on_device_geometry_vs_reference_golden(monkeypatch, name):
    """Every propagation level on on-device geometry (what cfg 5 does on
    levels 4-5): node tables from otf_tables_kernel per chunk of parent rows
    (libdevice acos / atan2 / sincos instead of the host's numpy values),
    still within the north-star tolerance of the reference's output."""
    _have(name)
    if not plan_matches_golden(name):
        pytest.skip("host numpy produced a different plan than the golden host")
    monkeypatch.setenv("IFGFB_GEOM_ON_DEVICE", "all")
    monkeypatch.delenv("IFGFB_OTF_PRE_MB", raising=False)
    z, inp = golden(name), inputs(name)
    op = MullerOperator(inp["disc"], inp["mats"], inp["smap"], inp["moments"],
                        (inp["corr"].ell_idx, inp["corr"].src_idx), tree=inp["tree"],
                        hierarchy=inp["hier"])
    assert sorted(op.plan.otf_levels) == list(range(4, inp["tree"].depth + 1))
    assert rel(op.apply(z["y"]), z["apply_y"]) < 1e-10


@pytest.mark.parametrize("name", ["s1", "c1", "c2n4", "c2n8"])
def test_potentials_vs_reference_golden(name):
    _have(name)
    if not plan_matches_golden(name):
        pytest.skip("host numpy produced a different plan than the golden host")
    z = golden(name)
    op = device_op(name)
    m, j = op.decode(z["y"])
    s, d = op.potentials(DensityBlock.from_currents(op.disc, j, m))
    rows = golden_rows(name)
    assert rel(s[..., rows], z["s_val"]) < 1e-13
    assert rel(d[..., rows], z["d_val"]) < 1e-9


def test_apply_vs_oracle_on_host():
    inp = inputs("s1")
    op = device_op("s1")
    y = np.random.default_rng(9).normal(size=(op.n_unknowns, 2)) @ [1, 1j]
    ref = oracle.muller_apply(oracle.OperatorData(
        inp["disc"], inp["mats"], inp["smap"], inp["moments"],
        inp["corr"].ell_idx, inp["corr"].src_idx, inp["tree"], inp["hier"]), y)
    assert rel(op.apply(y), ref) < 1e-10


@pytest.mark.parametrize("n_c", [13, 16])
def test_apply_high_patch_order_vs_oracle(n_c):
    """n_c = 13..16: the per-patch kernels (K1 packing, K7 assembly) need more
    than the default 48 KB of dynamic shared memory (20 n_c^2 and 16 n_c^2
    complex values); sphere(1, n_c) against the oracle on this host."""
    from paper_2408_02274_b200 import nearfield, octree, surface
    from paper_2408_02274_b200.operator import MaterialPair
    disc = surface.make_sphere_surface(1, n_c)
    mats = MaterialPair(1.0, 1.0, 2.25, 1.0, 2 * np.pi)
    tree = octree.build_box_tree(disc.points, max(abs(mats.kappa_e), abs(mats.kappa_i)))
    hier = octree.build_cone_hierarchy(tree)
    smap = nearfield.classify_targets(disc)
    mom = nearfield.compute_moments(disc, smap, nearfield.SingularQuadratureConfig(),
                                    mats.kappas)
    cp = nearfield.correction_pairs(disc, tree, smap)
    op = MullerOperator(disc, mats, smap, mom, (cp.ell_idx, cp.src_idx), tree=tree,
                        hierarchy=hier)
    y = np.random.default_rng(n_c).normal(size=(op.n_unknowns, 2)) @ [1, 1j]
    ref = oracle.muller_apply(oracle.OperatorData(
        disc, mats, smap, mom, cp.ell_idx, cp.src_idx, tree, hier), y)
    assert rel(op.apply(y), ref) < 1e-10


def test_device_and_host_paths_bitwise_equal_and_deterministic():
    op = device_op("c1")
    y = golden("c1")["y"]
    a = op.apply(y)
    b = op.apply(y)
    yd = torch.from_numpy(y).cuda()
    c = op.apply_device(yd).cpu().numpy()
    assert np.array_equal(a, b) and np.array_equal(a, c)


def test_apply_linearity():
    op = device_op("c1")
    rng = np.random.default_rng(2)
    n = op.n_unknowns
    y1 = rng.normal(size=n) + 1j * rng.normal(size=n)
    y2 = rng.normal(size=n) + 1j * rng.normal(size=n)
    lhs = op.apply(0.7 * y1 - 1.3j * y2)
    rhs = 0.7 * op.apply(y1) - 1.3j * op.apply(y2)
    # reference's own linearity residual here is 5.4e-11 (golden floor)
    assert rel(lhs, rhs) < 2e-10


def test_apply_rejects_wrong_length():
    op = device_op("s1")
    with pytest.raises(ValueError):
        op.apply(np.zeros(op.n_unknowns + 1, complex))


def test_gmres_matches_reference_history():
    if not plan_matches_golden("c1"):
        pytest.skip("host numpy produced a different plan than the golden host")
    z = golden("c1_gmres")
    op = device_op("c1")
    k0 = 2 * np.pi
    b = op.rhs(plane_wave(k0, direction=(0.0, 0.0, 1.0),
                          polarization=(1.0, 0.0, 0.0), omega=k0))
    assert np.array_equal(b, z["b"])
    x, rep = gmres(op, b, tol=1e-6, max_iter=300)
    ref = z["residuals"]
    assert rep.converged and rep.iterations == int(z["iterations"]) == 38
    r = np.array(rep.residuals)
    # north star: history matches to 1e-8 (the residuals are already
    # normalised by ||b||).  Per entry, relative: matvec noise at the
    # reference's own floor (1e-10, its D_far vec/seq level) moves the
    # history by 1.2e-8 (tools/gmres_sensitivity.py), so 5e-8 relative.
    assert np.max(np.abs(r - ref)) < 1e-8
    assert np.max(np.abs(r - ref) / ref) < 5e-8
    assert rel(x, z["x"]) < 1e-8
    assert np.linalg.norm(b - op.apply(x)) / np.linalg.norm(b) <= 2e-6


def test_gmres_basis_spill_to_host_is_bitwise_equal():
    """Krylov basis chunks in pinned host memory (forced by an unreachable
    device reserve) give the identical iteration: same kernels, same order,
    rows read over PCIe instead of HBM."""
    op = device_op("c1")
    k0 = 2 * np.pi
    b = op.rhs(plane_wave(k0, direction=(0.0, 0.0, 1.0),
                          polarization=(1.0, 0.0, 0.0), omega=k0))
    x1, r1 = gmres(op, b, tol=1e-6, max_iter=300)
    x2, r2 = gmres(op, b, tol=1e-6, max_iter=300, basis_device_reserve=1 << 60)
    assert r2.basis_host_rows > r2.iterations and r1.basis_host_rows == 0
    assert r1.residuals == r2.residuals
    assert np.array_equal(x1, x2)


def test_gmres_generic_callables():
    rng = np.random.default_rng(1)
    b = rng.normal(size=20) + 1j * rng.normal(size=20)
    x, rep = gmres(lambda v: v, b, tol=1e-12)
    assert rep.iterations == 1 and rep.converged and np.abs(x - b).max() < 1e-12
    x, rep = gmres(lambda v: 2 * v, np.zeros(10, complex), tol=1e-10)
    assert rep.iterations == 0 and rep.converged and not x.any()
    n = 60
    a = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n)) + 5 * np.eye(n)
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    x, rep = gmres(lambda v: a @ v, b, tol=1e-10, max_iter=n)
    assert np.all(np.diff(rep.residuals) <= 1e-14)
    assert np.abs(x - np.linalg.solve(a, b)).max() < 1e-8
    x, rep = gmres(lambda v: a @ v, b, tol=1e-30, max_iter=5)
    assert not rep.converged and rep.iterations == 5
    with pytest.raises(ValueError):
        gmres(lambda v: v, b, tol=0.0)


@pytest.mark.parametrize("name", ["s1", "c1"])
def test_geometry_on_device_matches_reference(name):
    """Memory-lean plan: node geometry and re-centering ratios computed in
    the propagation kernel (large configurations) instead of per-type
    tables.  Same sigma assignment, continuous values within a few ulps:
    the raw far field meets the same 1e-13 bar as the table path and the
    apply the 1e-10 parity bar (D_far amplifies ulp differences by 1/h)."""
    if not plan_matches_golden(name):
        pytest.skip("host numpy produced a different plan than the golden host")
    from paper_2408_02274_b200.engine import FarFieldPlan
    inp, z = inputs(name), golden(name)
    plan = FarFieldPlan(inp["tree"], inp["hier"], inp["disc"].normals, 1e-6,
                        kappas=inp["kappas"], geometry_on_device="all")
    assert plan.otf_levels == set(range(4, inp["tree"].depth + 1))
    dev = torch.device("cuda")
    w = torch.from_numpy(np.ascontiguousarray(z["weights"])).to(dev)
    out = torch.empty((w.shape[0], 2, w.shape[1]), dtype=torch.complex128, device=dev)
    od = torch.empty_like(out)
    plan.far_apply_device(w, inp["kappas"], out, od)
    assert rel(out.cpu().numpy(), z["far"]) < 1e-13
    assert rel(od.cpu().numpy(), z["far_disp"]) < 1e-13
    op = MullerOperator(
        inp["disc"], inp["mats"], inp["smap"], inp["moments"],
        (inp["corr"].ell_idx, inp["corr"].src_idx), tree=inp["tree"],
        hierarchy=inp["hier"], geometry_on_device="all")
    assert rel(op.apply(z["y"]), z["apply_y"]) < 1e-10


def test_gmres_slab_matches_reference_history():
    """Short cfg-4-like slab (sl1, eps_r 12.11): the device GMRES history
    for a broadside plane wave follows the reference's (15 iterations; the
    high-contrast thin body converges slowly in the reference too)."""
    if not plan_matches_golden("sl1"):
        pytest.skip("host numpy produced a different plan than the golden host")
    z = golden("sl1_gmres")
    op = device_op("sl1")
    k0 = float(op.materials.omega)
    b = op.rhs(plane_wave(k0, direction=(0.0, 1.0, 0.0),
                          polarization=(0.0, 0.0, 1.0), omega=k0))
    assert rel(b, z["b"]) < 1e-14
    x, rep = gmres(op, b, tol=1e-12, max_iter=15)
    r = np.array(rep.residuals)
    assert r.size == z["residuals"].size
    assert np.max(np.abs(r - z["residuals"])) < 1e-7
    assert rel(x, z["x"]) < 1e-6
