"""The CPU oracle pinned against golden vectors of the unmodified reference,
and against direct sums / analytic answers (reference tests/test_ifgf.py,
tests/test_solver.py restated)."""

import numpy as np
import pytest

import oracle
from _support import golden, inputs, rel
from paper_2408_02274_b200.octree import build_box_tree, build_cone_hierarchy


def naive_far(tree, w, kappas):
    d = tree.depth
    coords = tree.level(d).coords[tree.point_boxes(d)]
    wt = np.atleast_2d(w)[:, tree.perm]
    n = tree.points.shape[0]
    out = np.zeros((wt.shape[0], len(kappas), n), dtype=complex)
    for ell in range(n):
        t = tree.iperm[ell]
        far = np.abs(coords - coords[t]).max(axis=1) >= 2
        r = np.linalg.norm(tree.points[t] - tree.points[far], axis=1)
        for k, kap in enumerate(kappas):
            out[:, k, ell] = (np.exp(1j * kap * r) / (4 * np.pi * r) * wt[:, far]).sum(1)
    return out


def test_oracle_far_field_vs_reference_golden():
    z, inp = golden("rand_ifgf"), inputs("rand_ifgf")
    out, od = oracle.far_field(inp["tree"], inp["hier"], z["weights"],
                               inp["kappas"], inp["disc"].normals, 1e-6)
    assert rel(out, z["far"]) < 1e-13
    assert rel(od, z["far_disp"]) < 1e-13


def test_oracle_apply_vs_reference_golden():
    z, inp = golden("s1"), inputs("s1")
    op = oracle.OperatorData(inp["disc"], inp["mats"], inp["smap"],
                             inp["moments"], inp["corr"].ell_idx,
                             inp["corr"].src_idx, inp["tree"], inp["hier"])
    out = oracle.muller_apply(op, z["y"])
    # 1e-10 is the north-star bar; the reference's own vec/seq floor here is
    # 5.0e-11 (golden floor_vec_seq_apply)
    assert rel(out, z["apply_y"]) < 1e-10


def test_oracle_apply_superellipsoid_vs_reference_golden():
    """Non-sphere geometry (BASELINE cfg 3's body, PATCHGRID loaded by both
    sides).  The reference's own linearity floor here is 1.5e-10
    (golden floor_linearity), so the bar is 3e-10."""
    z, inp = golden("se1"), inputs("se1")
    op = oracle.OperatorData(inp["disc"], inp["mats"], inp["smap"],
                             inp["moments"], inp["corr"].ell_idx,
                             inp["corr"].src_idx, inp["tree"], inp["hier"])
    assert float(z["floor_linearity"]) < 3e-10
    assert rel(oracle.muller_apply(op, z["y"]), z["apply_y"]) < 3e-10


def test_oracle_apply_slab_vs_reference_golden():
    """Short cfg-4-like slab (exponent-8 superellipsoid 2 x 0.25 x 0.11
    wavelengths, eps_r 12.11), PATCHGRID loaded by both sides."""
    z, inp = golden("sl1"), inputs("sl1")
    op = oracle.OperatorData(inp["disc"], inp["mats"], inp["smap"],
                             inp["moments"], inp["corr"].ell_idx,
                             inp["corr"].src_idx, inp["tree"], inp["hier"])
    assert rel(oracle.muller_apply(op, z["y"]), z["apply_y"]) < 1e-10


def test_oracle_two_level_toy_matches_dense():
    rng = np.random.default_rng(4)
    src = rng.normal(size=(20, 3)) * 0.05 + [0.1, 0.1, 0.1]
    tgt = rng.normal(size=(20, 3)) * 0.05 + [0.9, 0.85, 0.9]
    pts = np.vstack([src, tgt])
    tree = build_box_tree(pts, 6.0)
    hier = build_cone_hierarchy(tree)
    w = np.zeros((1, 40), dtype=complex)
    w[0, :20] = rng.normal(size=20) + 1j * rng.normal(size=20)
    out, _ = oracle.far_field(tree, hier, w, (6.0,))
    ref = naive_far(tree, w, (6.0,))
    nz = np.abs(ref) > 1e-13
    assert np.abs(out[nz] - ref[nz]).max() < 1e-4 * np.abs(ref[nz]).max()


def test_oracle_self_interaction_excluded():
    pts = np.array([[0.05, 0.05, 0.05], [0.95, 0.95, 0.95]])
    tree = build_box_tree(pts, 40.0)
    hier = build_cone_hierarchy(tree)
    out, _ = oracle.far_field(tree, hier, np.array([[1.0 + 0j, 0.0]]), (40.0,))
    r = np.linalg.norm(pts[1] - pts[0])
    assert abs(out[0, 0, 0]) < 1e-12
    assert out[0, 0, 1] == pytest.approx(np.exp(1j * 40 * r) / (4 * np.pi * r), rel=2e-4)


def test_oracle_gmres_basics():
    rng = np.random.default_rng(1)
    b = rng.normal(size=20) + 1j * rng.normal(size=20)
    x, k, hist, ok, _ = oracle.gmres(lambda v: v, b, tol=1e-12)
    assert k == 1 and ok and np.abs(x - b).max() < 1e-12
    n = 50
    a = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n)) + n * np.eye(n)
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    x, k, hist, ok, _ = oracle.gmres(lambda v: a @ v, b, tol=1e-12, max_iter=n)
    ref = np.linalg.solve(a, b)
    assert ok and np.abs(x - ref).max() < 1e-10 * np.abs(ref).max()
    assert np.all(np.diff(hist) <= 1e-14)
    x, k, hist, ok, _ = oracle.gmres(lambda v: 2 * v, np.zeros(10, complex), tol=1e-10)
    assert k == 0 and ok and np.all(x == 0)
