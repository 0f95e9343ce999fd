"""GPU far field (ifgfb_far_apply through the drop-in ``ifgf_apply``) against
the reference golden vectors, the oracle run on this host, and the
reference's own far-field tests (tests/test_ifgf.py:225-389) restated."""

import numpy as np
import pytest

import oracle
from _support import (GOLDEN, golden, golden_rows, golden_weights, inputs,
                      plan_matches_golden, rel)
from paper_2408_02274_b200 import surface
from paper_2408_02274_b200.engine import ifgf_apply
from paper_2408_02274_b200.octree import build_box_tree, build_cone_hierarchy

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["rand_ifgf", "s1", "c1", "c2n4", "c2n8"])
def test_far_field_vs_reference_golden(name):
    if not (GOLDEN / f"{name}.npz").exists():
        pytest.skip(f"{name} fixture not generated")
    if name != "rand_ifgf" and not plan_matches_golden(name):
        pytest.skip("host numpy produced a different plan than the golden host")
    z, inp = golden(name), inputs(name)
    out, od = ifgf_apply(inp["tree"], inp["hier"], golden_weights(name), inp["kappas"],
                         displaced_normals=inp["disc"].normals,
                         displaced_step=1e-6)
    rows = golden_rows(name)
    # reference floor for ifgf outputs: vec vs seq 9.6e-16
    assert rel(out[..., rows], z["far"]) < 1e-13
    assert rel(od[..., rows], z["far_disp"]) < 1e-13


def test_far_field_vs_oracle_on_host():
    z, inp = golden("rand_ifgf"), inputs("rand_ifgf")
    w = np.random.default_rng(11).normal(size=(3, inp["disc"].n_points)) * (1 + 0.5j)
    got, gd = ifgf_apply(inp["tree"], inp["hier"], w, inp["kappas"],
                         displaced_normals=inp["disc"].normals)
    ref, rd = oracle.far_field(inp["tree"], inp["hier"], w, inp["kappas"],
                               inp["disc"].normals, 1e-6)
    assert rel(got, ref) < 1e-13 and rel(gd, rd) < 1e-13


def test_channel_independence_and_linearity():
    disc = surface.make_sphere_surface(1, 10)
    kap = (np.pi, 1.3 * np.pi)
    tree = build_box_tree(disc.points, max(kap))
    hier = build_cone_hierarchy(tree)
    n = disc.n_points
    rng = np.random.default_rng(6)
    w = np.zeros((4, n), dtype=complex)
    w[2] = rng.normal(size=n) + 1j * rng.normal(size=n)
    out, _ = ifgf_apply(tree, hier, w, kap)
    assert np.abs(out[[0, 1, 3]]).max() == 0.0
    assert np.abs(out[2]).max() > 0.0
    w2 = np.zeros_like(w)
    w2[2] = rng.normal(size=n)
    a, _ = ifgf_apply(tree, hier, w + 0.5j * w2, kap)
    b, _ = ifgf_apply(tree, hier, w, kap)
    c, _ = ifgf_apply(tree, hier, w2, kap)
    assert np.abs(a - b - 0.5j * c).max() < 1e-12 * np.abs(a).max()


def test_vec_seq_identical_and_deterministic():
    disc = surface.make_sphere_surface(2, 8)
    kap = (np.pi, 2 * np.pi)
    tree = build_box_tree(disc.points, max(kap))
    hier = build_cone_hierarchy(tree)
    w = np.random.default_rng(7).normal(size=(3, disc.n_points)) * (1 - 1j)
    v, _ = ifgf_apply(tree, hier, w, kap, mode="vec")
    s, _ = ifgf_apply(tree, hier, w, kap, mode="seq")
    v2, _ = ifgf_apply(tree, hier, w, kap, mode="vec")
    assert np.abs(v - s).max() < 1e-12 * np.abs(v).max()
    assert np.array_equal(v, v2)          # bitwise run-to-run
    with pytest.raises(ValueError):
        ifgf_apply(tree, hier, w, kap, mode="bogus")


def test_many_channels_and_three_kernels():
    """nch*nk > 16 columns: processed as column groups on device."""
    inp = inputs("rand_ifgf")
    n = inp["disc"].n_points
    rng = np.random.default_rng(3)
    w = rng.normal(size=(11, n)) + 1j * rng.normal(size=(11, n))
    kap = (2 * np.pi, 3 * np.pi, 2.5 * np.pi)
    got, _ = ifgf_apply(inp["tree"], inp["hier"], w, kap)
    ref, _ = oracle.far_field(inp["tree"], inp["hier"], w, kap)
    assert got.shape == (11, 3, n)
    assert rel(got, ref) < 1e-13


def test_self_interaction_excluded():
    pts = np.array([[0.05, 0.05, 0.05], [0.95, 0.95, 0.95]])
    tree = build_box_tree(pts, 40.0)
    hier = build_cone_hierarchy(tree)
    out, _ = ifgf_apply(tree, hier, np.array([[1.0 + 0j, 0.0]]), (40.0,))
    r = np.linalg.norm(pts[1] - pts[0])
    assert abs(out[0, 0, 0]) < 1e-12
    assert out[0, 0, 1] == pytest.approx(np.exp(1j * 40 * r) / (4 * np.pi * r), rel=2e-4)


def test_shallow_tree_gives_zero_far_field():
    pts = np.random.default_rng(1).normal(size=(30, 3)) * 0.01
    tree = build_box_tree(pts, 1.0)
    hier = build_cone_hierarchy(tree)
    out, od = ifgf_apply(tree, hier, np.ones((2, 30)), (1.0, 2.0),
                         displaced_normals=np.ones((30, 3)))
    assert out.shape == (2, 2, 30) and not out.any() and not od.any()


def test_sphere_accuracy_vs_naive_far_sums():
    from test_oracle import naive_far
    disc = surface.make_sphere_surface(2, 12)
    kap = (2 * np.pi, 3 * np.pi)
    tree = build_box_tree(disc.points, max(kap))
    hier = build_cone_hierarchy(tree)
    rng = np.random.default_rng(5)
    w = rng.normal(size=(2, disc.n_points)) + 1j * rng.normal(size=(2, disc.n_points))
    out, _ = ifgf_apply(tree, hier, w, kap)
    idx = rng.choice(disc.n_points, 150, replace=False)
    sub = np.zeros(disc.n_points, bool)
    sub[idx] = True
    ref = naive_far(tree, w, kap)
    assert rel(out[:, :, idx], ref[:, :, idx]) < 1.5e-4


def test_displaced_outputs_fd_vs_analytic():
    disc = surface.make_sphere_surface(1, 10)
    kappa = np.pi
    tree = build_box_tree(disc.points, kappa)
    hier = build_cone_hierarchy(tree)
    rng = np.random.default_rng(8)
    w = rng.normal(size=(1, disc.n_points)) + 1j * rng.normal(size=(1, disc.n_points))
    h = 1e-6
    out, od = ifgf_apply(tree, hier, w, (kappa,), displaced_normals=disc.normals,
                         displaced_step=h)
    fd = (od - out) / h
    d = tree.depth
    coords = tree.level(d).coords[tree.point_boxes(d)]
    wt = w[:, tree.perm]
    for ell in rng.choice(disc.n_points, 30, replace=False):
        t = tree.iperm[ell]
        far = np.abs(coords - coords[t]).max(axis=1) >= 2
        dx = tree.points[t] - tree.points[far]
        r = np.linalg.norm(dx, axis=1)
        q = (dx @ disc.normals[ell]) * (1j * kappa * r - 1) * np.exp(1j * kappa * r) / (4 * np.pi * r**3)
        ref = (q * wt[0, far]).sum()
        if abs(ref) > 1e-3:
            assert fd[0, 0, ell] == pytest.approx(ref, rel=2e-3)


def _naive_far_at(tree, w, kappas, targets):
    """Direct far sums (reference naive_far_sums, test_ifgf.py:22-38) at a
    subset of targets (original indices): sources outside the target's
    finest-level neighbour boxes."""
    d = tree.depth
    coords = tree.level(d).coords[tree.point_boxes(d)]
    wt = np.atleast_2d(w)[:, tree.perm]
    out = np.zeros((wt.shape[0], len(kappas), len(targets)), dtype=complex)
    for j, ell in enumerate(targets):
        t = tree.iperm[ell]
        far = np.abs(coords - coords[t]).max(axis=1) >= 2
        r = np.linalg.norm(tree.points[t] - tree.points[far], axis=1)
        for k, kap in enumerate(kappas):
            out[:, k, j] = (np.exp(1j * kap * r) / (4 * np.pi * r) * wt[:, far]).sum(1)
    return out


@pytest.mark.parametrize("geometry", ["sphere8", "superellipsoid_cfg3"])
def test_full_size_accuracy_linearity_determinism(geometry):
    """BASELINE sizes, size-independent properties: the far field against
    direct sums at 100 sampled targets within the reference's accuracy bar
    (test_ifgf.py:296-308, 1.5e-4), linearity to 1e-12 (test_ifgf.py:
    311-330) and bitwise run-to-run determinism.  sphere8 = cfg 2 at
    n = 8 (k0 = 8 pi, 153,600 unknowns, depth 7); superellipsoid_cfg3 =
    cfg 3 (221,184 unknowns, depth 8)."""
    if geometry == "sphere8":
        disc = surface.make_sphere_surface(8, 10)
        kap = (8 * np.pi, 12 * np.pi)
    else:
        disc = surface.make_superellipsoid_surface(8, 12, (2.0, 1.0, 0.5), 4.0)
        kap = (4 * np.pi, 8 * np.pi)
    tree = build_box_tree(disc.points, max(kap))
    hier = build_cone_hierarchy(tree)
    n = disc.n_points
    rng = np.random.default_rng(7)
    w = rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n))
    w2 = rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n))
    a, _ = ifgf_apply(tree, hier, w, kap)
    a2, _ = ifgf_apply(tree, hier, w, kap)
    assert np.array_equal(a, a2)
    idx = rng.choice(n, 100, replace=False)
    assert rel(a[:, :, idx], _naive_far_at(tree, w, kap, idx)) < 1.5e-4
    b, _ = ifgf_apply(tree, hier, w2, kap)
    c, _ = ifgf_apply(tree, hier, w + 0.5j * w2, kap)
    assert np.abs(c - a - 0.5j * b).max() < 1e-12 * np.abs(c).max()


def test_displaced_point_across_phi_seam():
    """Displaced points (x + h n) that cross the phi = 0 seam of a source
    box's cone stay on the undisplaced point's branch (octree.emission_plan;
    the reference takes phi mod 2 pi there and extrapolates the angular
    polynomial by ~2 n_a intervals, see DESIGN 2).  A large step makes many
    crossings; the displaced far field must match direct sums at x + h n."""
    disc = surface.make_sphere_surface(2, 10)
    kap = (2 * np.pi, 3 * np.pi)
    tree = build_box_tree(disc.points, max(kap))
    hier = build_cone_hierarchy(tree)
    step = 2e-3
    rng = np.random.default_rng(4)
    w = rng.normal(size=(1, disc.n_points)) + 1j * rng.normal(size=(1, disc.n_points))
    out, od = ifgf_apply(tree, hier, w, kap, displaced_normals=disc.normals,
                         displaced_step=step)
    # targets whose displacement crosses a seam at some level
    from paper_2408_02274_b200.octree import cone_coords
    disp = tree.points + step * disc.normals[tree.perm]
    cross = set()
    for d in range(3, tree.depth + 1):
        cl, lvl = hier.level(d), tree.level(d)
        if cl.cpt_idx.size == 0:
            continue
        box = np.repeat(np.arange(lvl.n_boxes), np.diff(cl.cpt_off))
        ctr = lvl.centers[box]
        ph = cone_coords(tree.points[cl.cpt_idx] - ctr, np.zeros(3), lvl.side)[2]
        pd = cone_coords(disp[cl.cpt_idx] - ctr, np.zeros(3), lvl.side)[2]
        cross.update(int(tree.perm[t]) for t in cl.cpt_idx[np.abs(pd - ph) > np.pi])
    idx = np.array(sorted(cross))[:40]
    assert idx.size >= 5
    # direct far sums at x + h n with x's own far-box set
    dd = tree.depth
    coords = tree.level(dd).coords[tree.point_boxes(dd)]
    wt = w[:, tree.perm]
    ref = np.zeros((1, 2, idx.size), dtype=complex)
    for j, ell in enumerate(idx):
        t = tree.iperm[ell]
        far = np.abs(coords - coords[t]).max(axis=1) >= 2
        r = np.linalg.norm(disp[t] - tree.points[far], axis=1)
        for k, kp in enumerate(kap):
            ref[:, k, j] = (np.exp(1j * kp * r) / (4 * np.pi * r) * wt[:, far]).sum(1)
    assert rel(od[:, :, idx], ref) < 1e-3


@pytest.mark.parametrize("geometry_on_device", ["none", "all"])
def test_tile_free_propagation_is_bitwise_tile_records(monkeypatch, geometry_on_device):
    """Plans without MMA tile records (tiles formed in the propagation
    kernel from the nodes' sigma groups, the default) give bitwise the
    result of plans carrying ifgfb_row_tiles_fill's records."""
    from paper_2408_02274_b200.engine import FarFieldPlan
    inp, z = inputs("c1"), golden("c1")
    outs = []
    for mode in ("l1", "l1free"):
        monkeypatch.setenv("IFGFB_K4", mode)
        plan = FarFieldPlan(inp["tree"], inp["hier"], inp["disc"].normals, 1e-6,
                            kappas=inp["kappas"], geometry_on_device=geometry_on_device)
        import torch
        dev = torch.device("cuda")
        w = torch.from_numpy(np.ascontiguousarray(z["weights"])).to(dev)
        out = torch.empty((w.shape[0], 2, w.shape[1]), dtype=torch.complex128, device=dev)
        od = torch.empty_like(out)
        plan.far_apply_device(w, inp["kappas"], out, od)
        outs.append((out.cpu().numpy(), od.cpu().numpy(), plan.device_bytes()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert outs[1][2] < outs[0][2]        # no tile records on the device


@pytest.mark.parametrize("geometry_on_device", ["none", "all"])
@pytest.mark.parametrize("case", ["c1", "rand"])
def test_wide_warp_propagation_is_bitwise_five_warp(monkeypatch, geometry_on_device, case):
    """The wide-warp propagation kernel (IFGFB_K4=wide: 3 owner warps per
    parent row, up to 4 MMA row tiles of one sigma group sharing each B
    fragment load) performs the 5-warp kernel's per-node arithmetic in the
    same order: the far field is bitwise equal (2 kernels at c1, the
    1-kernel instantiation on the random 2-channel case)."""
    import torch
    from paper_2408_02274_b200.engine import FarFieldPlan
    if case == "c1":
        inp, z = inputs("c1"), golden("c1")
        tree, hier, normals, kappas, w_h = (inp["tree"], inp["hier"], inp["disc"].normals,
                                            inp["kappas"], z["weights"])
    else:
        from paper_2408_02274_b200 import octree, surface
        disc = surface.make_sphere_surface(2, 6)
        kappas = (3 * np.pi,)
        tree = octree.build_box_tree(disc.points, max(kappas))
        hier = octree.build_cone_hierarchy(tree)
        rng = np.random.default_rng(11)
        w_h = rng.normal(size=(5, disc.n_points)) + 1j * rng.normal(size=(5, disc.n_points))
        normals = disc.normals
    outs = []
    for mode in ("l1free", "wide"):
        monkeypatch.setenv("IFGFB_K4", mode)
        plan = FarFieldPlan(tree, hier, normals, 1e-6, kappas=kappas,
                            geometry_on_device=geometry_on_device)
        dev = torch.device("cuda")
        w = torch.from_numpy(np.ascontiguousarray(w_h)).to(dev)
        out = torch.empty((w.shape[0], len(kappas), w.shape[1]), dtype=torch.complex128,
                          device=dev)
        od = torch.empty_like(out)
        plan.far_apply_device(w, kappas, out, od)
        outs.append((out.cpu().numpy(), od.cpu().numpy()))
    assert np.isfinite(outs[1][0]).all() and np.abs(outs[1][0]).max() > 0
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("case", ["c1", "rand"])
def test_node_table_prepass_equals_in_kernel_geometry(monkeypatch, case):
    """On-device-geometry levels: the node tables tabulated per (instance,
    node) by otf_tables_kernel ahead of each propagation launch (default; in
    chunks of parent rows that fit the scratch) give the far field of the
    geometry computed inside the propagation kernel (IFGFB_OTF_PRE_MB=0);
    the chunking itself is bitwise neutral."""
    import torch
    from paper_2408_02274_b200.engine import FarFieldPlan
    if case == "c1":
        inp, z = inputs("c1"), golden("c1")
        tree, hier, normals, kappas, w_h = (inp["tree"], inp["hier"], inp["disc"].normals,
                                            inp["kappas"], z["weights"])
    else:
        from paper_2408_02274_b200 import octree, surface
        disc = surface.make_sphere_surface(2, 6)
        kappas = (3 * np.pi,)
        tree = octree.build_box_tree(disc.points, max(kappas))
        hier = octree.build_cone_hierarchy(tree)
        rng = np.random.default_rng(12)
        w_h = rng.normal(size=(5, disc.n_points)) + 1j * rng.normal(size=(5, disc.n_points))
        normals = disc.normals
    monkeypatch.setenv("IFGFB_K4", "wide")
    outs = []
    for env in ({"IFGFB_OTF_PRE_MB": "0"}, {}, {"IFGFB_OTF_PRE_INST": "40"}):
        for k in ("IFGFB_OTF_PRE_MB", "IFGFB_OTF_PRE_INST"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        plan = FarFieldPlan(tree, hier, normals, 1e-6, kappas=kappas, geometry_on_device="all")
        dev = torch.device("cuda")
        w = torch.from_numpy(np.ascontiguousarray(w_h)).to(dev)
        out = torch.empty((w.shape[0], len(kappas), w.shape[1]), dtype=torch.complex128,
                          device=dev)
        od = torch.empty_like(out)
        plan.far_apply_device(w, kappas, out, od)
        plan.far_apply_device(w, kappas, out, od)     # scratch reused across applies
        outs.append((out.cpu().numpy(), od.cpu().numpy(), plan.device_bytes()))
    assert np.isfinite(outs[1][0]).all() and np.abs(outs[1][0]).max() > 0
    assert outs[1][2] > outs[0][2]                    # the scratch is part of the plan
    assert np.array_equal(outs[1][0], outs[2][0]) and np.array_equal(outs[1][1], outs[2][1])
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
