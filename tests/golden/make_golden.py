"""Generate golden fixtures from the UNMODIFIED reference (`emscat`, imported
read-only from /root/reference/pkg/src).  Runs only in the build container;
the committed .npz outputs travel to the GPU hosts.

Usage:  python tests/golden/make_golden.py [s1] [c1] [c1gmres] [rand]

Fixtures (complex arrays stored as complex128):
  <name>.npz (s1, c1, se1, sl1, c2n4, c2n8)
    plan_digest_*   sha256 of every plan integer array (tree, cones,
                    accumulation types, emission rows, singular map,
                    correction lists) -- see plan_digests()
    y               matvec input, Re/Im iid N(0,1) from default_rng(0)
    apply_y         MullerOperator.apply(y)            (operators.py:399)
    weights         phi * disc.weights fed to ifgf_apply (operators.py:336)
    far / far_disp  ifgf_apply(..., mode='vec', normals, 1e-6)  (ifgf.py:885)
    rows            c2n4 / c2n8 only: the strided point subset at which
                    far, far_disp, s_val, d_val are stored (weights omitted;
                    they follow from y)
    s_val / d_val   potentials(dens)                   (operators.py:321)
    floor_*         reference self-consistency floors (linearity, vec/seq)
  c1_gmres.npz      GMRES tol 1e-6, plane wave exp(i k0 z) x-pol (cfg 1)
  rand_ifgf.npz     ifgf_apply on random (2, N) weights, kappas (2pi, 3pi)
  fields.npz        off-surface fields (reference.py:285-347) on sphere(1,10)
                    with smooth random tangential currents; Mie series
                    (reference.py:240-269) coefficients and fields; dipole;
                    the validate-sphere check (cli.py:258-289) on the
                    reference's own cfg-1 GMRES solution (c1_gmres.npz)
"""

from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent

CONFIGS = {
    # name: (n_refine, n_c, k0 / pi, eps_r)
    "s1": (1, 10, 2.0, 2.25),
    "c1": (2, 10, 2.0, 2.25),
    # superellipsoid |x/2|^4 + |y|^4 + |z/0.5|^4 = 1 (BASELINE cfg 3's body at
    # 2a = 2 wavelengths, eps_r 4): 1 x 1 subpatch per face, n_c = 8
    "se1": (1, 8, 1.0, 4.0),
    # short cfg-4-like slab: exponent-8 superellipsoid, half-extents
    # 2 x 0.25 x 0.11 wavelengths (wavelength 1), eps_r 12.11, (4, 2, 1) splits
    "sl1": ((4, 2, 1), 10, 2.0, 12.11),
    # BASELINE cfg 2 sizes the reference can run here (k0 = pi * n_refine,
    # reference cli.py:300-307): the benchmarked family at 38,400 and
    # 153,600 unknowns
    "c2n4": (4, 10, 4.0, 2.25),
    "c2n8": (8, 10, 8.0, 2.25),
}
# large fixtures keep the per-point outputs (far, far_disp, potentials) on a
# strided subset of points only (the `rows` array); y and apply_y are full
ROW_STRIDE = {"c2n4": 3, "c2n8": 8}
# non-sphere geometries: PATCHGRID files written by the framework's
# generator (surface.make_superellipsoid_surface) and committed next to the
# fixtures; both the reference and the framework load the same file with
# their own load_surface (reference geometry.py:286-329)
GEOMETRY = {"se1": dict(semi_axes=(2.0, 1.0, 0.5), exponent=4.0),
            "sl1": dict(semi_axes=(2.0, 0.25, 0.11), exponent=8.0)}


def geometry_file(name):
    path = OUT / f"{name}.patchgrid"
    if not path.exists():
        sys.path.insert(0, str(OUT.parents[1]))
        from paper_2408_02274_b200 import surface as fs
        nr, nc = CONFIGS[name][:2]
        fs.write_surface(fs.make_superellipsoid_surface(nr, nc, **GEOMETRY[name]), path)
    return path


def _h(a) -> str:
    a = np.ascontiguousarray(np.asarray(a))
    return hashlib.sha256(a.tobytes()).hexdigest()[:32]


def plan_digests(tree, hier, accum_types_fn, smap, corr_ell, corr_src,
                 emission_rows_fn):
    """Digest dict shared by the generator (reference objects) and the tests
    (framework objects).  Integer arrays plus the float arrays that feed them
    (centres, node grids) are hashed."""
    out = {"depth": np.int64(tree.depth)}
    out["perm"] = _h(tree.perm.astype(np.int64))
    for d in range(1, tree.depth + 1):
        lvl = tree.level(d)
        for a in ("codes", "pt_start", "pt_count", "parent", "nbr_idx",
                  "nbr_off", "cousin_idx", "cousin_off", "centers"):
            v = getattr(lvl, a)
            out[f"L{d}_{a}"] = _h(v.astype(np.float64 if a == "centers"
                                           else np.int64))
    for d in sorted(hier.cone_levels):
        cl = hier.level(d)
        for a in ("seg_ids", "seg_off", "cpt_idx", "cpt_off"):
            out[f"C{d}_{a}"] = _h(getattr(cl, a).astype(np.int64))
        out[f"C{d}_emit_rows"] = _h(emission_rows_fn(d).astype(np.int64))
    for d in sorted(hier.cone_levels):
        if d - 1 not in hier.cone_levels:
            continue
        sig, bnd, sc, child, prow, crow, geo = accum_types_fn(d)
        for nm, v in (("sigma", sig), ("bounds", bnd), ("scatter", sc),
                      ("inst_child", child), ("inst_prow", prow),
                      ("inst_crow", crow)):
            out[f"A{d}_{nm}"] = _h(v.astype(np.int64))
        out[f"A{d}_geom"] = _h(geo.astype(np.float64))
    out["smap_offsets"] = _h(smap.offsets.astype(np.int64))
    out["smap_patch_ids"] = _h(smap.patch_ids.astype(np.int64))
    out["corr_ell"] = _h(np.asarray(corr_ell, np.int64))
    out["corr_src"] = _h(np.asarray(corr_src, np.int64))
    return out


def _ref_accum(ri, tree, hier):
    def fn(d):
        types = ri._accum_types(tree, hier, d)
        cat = lambda f: np.concatenate([f(t).ravel() for t in types])
        geo = np.concatenate([np.concatenate([t.xs, t.xt, t.xp, t.r_parent,
                                              t.r_child]) for t in types])
        return (cat(lambda t: t.sigma), cat(lambda t: t.bounds),
                cat(lambda t: t.scatter_rows), cat(lambda t: t.inst_child),
                cat(lambda t: t.inst_prow), cat(lambda t: t.inst_crow), geo)
    return fn


def _ref_emit_rows(ri, tree, hier):
    def fn(d):
        cl, lvl = hier.level(d), tree.level(d)
        tg = cl.cpt_idx
        box = np.repeat(np.arange(lvl.n_boxes), np.diff(cl.cpt_off))
        s, th, ph, _ = ri.cone_coords(tree.points[tg] - lvl.centers[box],
                                      np.zeros(3), lvl.side)
        return ri._seg_row_lookup(cl, box, cl.seg_index(s, th, ph))
    return fn


def random_y(n: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.normal(size=4 * n) + 1j * rng.normal(size=4 * n)


def build(name):
    sys.path.insert(0, REF)
    import emscat.geometry as rg
    import emscat.ifgf as ri
    from emscat.operators import (DensityBlock, MaterialPair,
                                  build_muller_operator)
    nr, nc, k0pi, eps = CONFIGS[name]
    k0 = k0pi * np.pi
    if name in GEOMETRY:
        disc = rg.load_surface(geometry_file(name), nc)
    else:
        disc = rg.make_sphere_surface(nr, nc)
    mats = MaterialPair(1.0, 1.0, eps, 1.0, k0)
    t0 = time.time()
    op = build_muller_operator(disc, mats)
    print(name, "build", time.time() - t0, flush=True)
    n = disc.n_points
    y = random_y(n)
    op.apply(y)                       # fill lazy caches
    t0 = time.time()
    ay = op.apply(y)
    t_apply = time.time() - t0
    print(name, "apply", t_apply, flush=True)
    m, j = op.decode(y)
    dens = DensityBlock.from_currents(disc, j, m)
    w = dens.values * disc.weights
    far, far_d = ri.ifgf_apply(op.tree, op.hierarchy, w, mats.kappas,
                               mode="vec", displaced_normals=disc.normals,
                               displaced_step=op.config.fd_step)
    s_val, d_val = op.potentials(dens)
    # reference noise floors
    rng = np.random.default_rng(1)
    y2 = rng.normal(size=4 * n) + 1j * rng.normal(size=4 * n)
    lin = op.apply(0.7 * y - 1.3j * y2) - (0.7 * ay - 1.3j * op.apply(y2))
    floor_lin = np.linalg.norm(lin) / np.linalg.norm(ay)
    cs = op.moments.corrections
    dig = plan_digests(op.tree, op.hierarchy, _ref_accum(ri, op.tree,
                                                          op.hierarchy),
                       op.smap, cs.ell_idx, cs.src_idx,
                       _ref_emit_rows(ri, op.tree, op.hierarchy))
    stride = ROW_STRIDE.get(name, 1)
    rows = np.arange(0, n, stride)
    sub = (lambda a: a) if stride == 1 else (lambda a: np.ascontiguousarray(a[..., rows]))
    payload = dict(y=y, apply_y=ay, far=sub(far), far_disp=sub(far_d),
                   s_val=sub(s_val), d_val=sub(d_val), floor_linearity=floor_lin,
                   t_apply_ref_container=t_apply,
                   config=np.array([nr if np.isscalar(nr) else 0, nc, k0pi, eps]))
    if stride == 1:
        payload["weights"] = w
    else:
        payload["rows"] = rows
    if name == "s1":
        op.config = type(op.config)(fd_step=op.config.fd_step, mode="seq")
        ay_seq = op.apply(y)
        payload["floor_vec_seq_apply"] = (np.linalg.norm(ay_seq - ay) /
                                          np.linalg.norm(ay))
    for k, v in dig.items():
        payload["plan_digest_" + k] = np.array(v)
    np.savez_compressed(OUT / f"{name}.npz", **payload)
    print(name, "floor_lin", floor_lin, flush=True)


def build_gmres():
    sys.path.insert(0, REF)
    import emscat.geometry as rg
    from emscat.operators import MaterialPair, build_muller_operator
    from emscat.reference import plane_wave
    from emscat.solver import gmres
    disc = rg.make_sphere_surface(2, 10)
    k0 = 2 * np.pi
    mats = MaterialPair(1.0, 1.0, 2.25, 1.0, k0)
    op = build_muller_operator(disc, mats)
    b = op.rhs(plane_wave(k0, direction=(0.0, 0.0, 1.0),
                          polarization=(1.0, 0.0, 0.0), omega=k0))
    t0 = time.time()
    x, rep = gmres(op.apply, b, tol=1e-6, max_iter=300)
    np.savez_compressed(OUT / "c1_gmres.npz", b=b, x=x,
                        residuals=np.array(rep.residuals),
                        iterations=rep.iterations, wall=time.time() - t0)
    print("gmres", rep.iterations, rep.residuals[-1], time.time() - t0)


def build_rand():
    sys.path.insert(0, REF)
    import emscat.geometry as rg
    import emscat.ifgf as ri
    disc = rg.make_sphere_surface(1, 6)
    kap = (2 * np.pi, 3 * np.pi)
    tree = ri.build_box_tree(disc.points, max(kap))
    hier = ri.build_cone_hierarchy(tree)
    rng = np.random.default_rng(5)
    w = rng.normal(size=(2, disc.n_points)) + 1j * rng.normal(
        size=(2, disc.n_points))
    out, out_d = ri.ifgf_apply(tree, hier, w, kap, mode="vec",
                               displaced_normals=disc.normals,
                               displaced_step=1e-6)
    np.savez_compressed(OUT / "rand_ifgf.npz", weights=w, far=out,
                        far_disp=out_d, kappas=np.array(kap),
                        config=np.array([1, 6]))
    print("rand done")


def build_sl1_gmres():
    """GMRES history on the short slab (sl1) for a plane wave along +y,
    z-polarised: 15 iterations (tol 1e-12 is never reached)."""
    sys.path.insert(0, REF)
    import emscat.geometry as rg
    from emscat.operators import MaterialPair, build_muller_operator
    from emscat.reference import plane_wave
    from emscat.solver import gmres
    nr, nc, k0pi, eps = CONFIGS["sl1"]
    disc = rg.load_surface(geometry_file("sl1"), nc)
    k0 = k0pi * np.pi
    mats = MaterialPair(1.0, 1.0, eps, 1.0, k0)
    op = build_muller_operator(disc, mats)
    b = op.rhs(plane_wave(k0, direction=(0.0, 1.0, 0.0),
                          polarization=(0.0, 0.0, 1.0), omega=k0))
    x, rep = gmres(op.apply, b, tol=1e-12, max_iter=15)
    np.savez_compressed(OUT / "sl1_gmres.npz", b=b, x=x,
                        residuals=np.array(rep.residuals))
    print("sl1 gmres", rep.residuals)


def build_fields():
    sys.path.insert(0, REF)
    import emscat.geometry as rg
    from emscat.operators import DensityBlock, MaterialPair, build_muller_operator
    from emscat.reference import (_layer_fields, electric_dipole, evaluate_fields,
                                  fibonacci_sphere, mie_solution, plane_wave)
    k0 = 2 * np.pi
    mats = MaterialPair(1.0, 1.0, 2.25, 1.0, k0)
    pay = {}
    # layer fields with smooth random tangential currents on sphere(1,10)
    disc = rg.make_sphere_surface(1, 10)
    rng = np.random.default_rng(11)
    n = disc.normals
    c = rng.normal(size=(4, 3)) + 1j * rng.normal(size=(4, 3))
    m = np.cross(n, c[0] + np.outer(disc.points[:, 2], c[1]))
    j = np.cross(n, c[2] + np.outer(disc.points[:, 0], c[3]))
    dens = DensityBlock.from_currents(disc, j, m)
    p_in = fibonacci_sphere(64, 0.6)
    p_out = 1.8 * fibonacci_sphere(64, 1.0)
    pay.update(s1_m=m, s1_j=j, s1_dens=dens.values, p_in=p_in, p_out=p_out,
               lf_in=_layer_fields(disc, dens, mats.kappa_i, p_in),
               lf_out=_layer_fields(disc, dens, mats.kappa_e, p_out))
    e_in, h_in = evaluate_fields(disc, dens, mats, p_in, "interior")
    inc = plane_wave(k0, omega=k0)
    e_out, h_out = evaluate_fields(disc, dens, mats, p_out, "exterior",
                                   incident=inc)
    pay.update(e_in=e_in, h_in=h_in, e_out=e_out, h_out=h_out)
    # Mie series
    mie = mie_solution(1.0, mats)
    pm_in = fibonacci_sphere(50, 0.7)
    pm_out = fibonacci_sphere(50, 1.5)
    ei, hi = mie.interior_fields(pm_in)
    es, hs = mie.exterior_scattered(pm_out)
    pay.update(mie_a=mie.a, mie_b=mie.b, mie_c=mie.c, mie_d=mie.d,
               pm_in=pm_in, pm_out=pm_out, mie_e_in=ei, mie_h_in=hi,
               mie_e_sc=es, mie_h_sc=hs)
    dip = electric_dipole([0.1, -0.2, 0.3], [1.0, 0.5j, -0.25], eps=2.0,
                          omega=k0)
    ed, hd = dip.fields(pm_out)
    pay.update(dip_e=ed, dip_h=hd)
    # validate-sphere on the reference's cfg-1 GMRES solution
    z = np.load(OUT / "c1_gmres.npz")
    disc1 = rg.make_sphere_surface(2, 10)
    op = build_muller_operator(disc1, mats)
    mm, jj = op.decode(z["x"])
    d1 = DensityBlock.from_currents(disc1, jj, mm)
    pv = fibonacci_sphere(1000, 0.7)
    e_num, h_num = evaluate_fields(disc1, d1, mats, pv, "interior")
    # c1_gmres is driven by exp(+i k0 z) x_hat (BASELINE cfg 1): that is the
    # series' own frame (MieSolution._eval), not the rotated -z default
    e_ref, h_ref = mie._eval(pv, "interior")
    pay.update(val_e=e_num, val_h=h_num,
               val_err_e=np.linalg.norm(e_num - e_ref) / np.linalg.norm(e_ref),
               val_err_h=np.linalg.norm(h_num - h_ref) / np.linalg.norm(h_ref))
    np.savez_compressed(OUT / "fields.npz", **pay)
    print("fields done", pay["val_err_e"], pay["val_err_h"])


if __name__ == "__main__":
    which = sys.argv[1:] or ["rand", "s1", "c1", "c1gmres", "fields"]
    for w_ in which:
        if w_ == "fields":
            build_fields()
        elif w_ == "sl1gmres":
            build_sl1_gmres()
        elif w_ == "c1gmres":
            build_gmres()
        elif w_ == "rand":
            build_rand()
        else:
            build(w_)
