"""Shared helpers for the test suite (golden fixtures, plan inputs)."""

from __future__ import annotations

import functools
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(GOLDEN))

from make_golden import plan_digests  # noqa: E402
from paper_2408_02274_b200 import nearfield, octree, surface  # noqa: E402
from paper_2408_02274_b200.operator import MaterialPair  # noqa: E402


def rel(a, b) -> float:
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) /
                 np.linalg.norm(np.asarray(b)))


@functools.lru_cache(maxsize=None)
def golden(name: str):
    return dict(np.load(GOLDEN / f"{name}.npz"))


@functools.lru_cache(maxsize=None)
def inputs(name: str):
    """Plan inputs built by the framework for a golden configuration."""
    z = golden(name)
    if name == "rand_ifgf":
        disc = surface.make_sphere_surface(1, 6)
        kap = tuple(float(k) for k in z["kappas"])
        tree = octree.build_box_tree(disc.points, max(kap))
        hier = octree.build_cone_hierarchy(tree)
        return dict(disc=disc, kappas=kap, tree=tree, hier=hier)
    nr, nc, k0pi, eps = z["config"]
    if (GOLDEN / f"{name}.patchgrid").exists():
        disc = surface.load_surface(GOLDEN / f"{name}.patchgrid", int(nc))
    else:
        disc = surface.make_sphere_surface(int(nr), int(nc))
    mats = MaterialPair(1.0, 1.0, float(eps), 1.0, float(k0pi) * np.pi)
    kmax = max(abs(mats.kappa_e), abs(mats.kappa_i))
    tree = octree.build_box_tree(disc.points, kmax)
    hier = octree.build_cone_hierarchy(tree)
    smap = nearfield.classify_targets(disc)
    mom = nearfield.compute_moments(disc, smap,
                                    nearfield.SingularQuadratureConfig(),
                                    mats.kappas)
    cp = nearfield.correction_pairs(disc, tree, smap)
    return dict(disc=disc, mats=mats, kappas=mats.kappas, tree=tree,
                hier=hier, smap=smap, moments=mom, corr=cp)


def framework_digests(inp) -> dict:
    """Digests of the framework plan in the reference's layout."""
    tree, hier = inp["tree"], inp["hier"]

    def accum(d):
        ap = octree.accumulation_plan(tree, hier, d)
        prow = np.searchsorted(ap.inst_off, np.arange(ap.n_instances),
                               side="right") - 1
        sig, bnd, sc, ch, pr, cr, geo = [], [], [], [], [], [], []
        order = np.lexsort((prow, ap.inst_child, ap.inst_type))
        starts = np.searchsorted(ap.inst_type[order], np.arange(ap.n_types))
        ends = np.append(starts[1:], order.size)
        for t in range(ap.n_types):
            g0, g1 = ap.sig_off[t], ap.sig_off[t + 1]
            gs = ap.group_bounds[g0:g1]
            # sigma = child segment id of each group (recomputed from crow)
            sel = order[starts[t]:ends[t]]
            crow = np.stack([ap.crow[ap.inst_crow_off[i]:ap.inst_crow_off[i + 1]]
                             for i in sel])
            sig.append(ap.group_sigma[g0:g1])
            bnd.append(np.append(gs, 75))
            sc.append(ap.scatter[t])
            ch.append(ap.inst_child[sel])
            pr.append(prow[sel])
            cr.append(crow.ravel())
            geo.append(np.concatenate([ap.xs[t], ap.xt[t], ap.xp[t],
                                       ap.r_parent[t], ap.r_child[t]]))
        cat = np.concatenate
        return cat(sig), cat(bnd), cat(sc), cat(ch), cat(pr), cat(cr), cat(geo)

    def emit_rows(d):
        return octree.emission_plan(tree, hier, d).row

    return plan_digests(tree, hier, accum, inp["smap"], inp["corr"].ell_idx,
                        inp["corr"].src_idx, emit_rows)


def golden_digests(name: str) -> dict:
    z = golden(name)
    return {k[len("plan_digest_"):]: (str(v) if v.dtype.kind == "U" else v)
            for k, v in z.items() if k.startswith("plan_digest_")}


def plan_matches_golden(name: str) -> bool:
    mine = framework_digests(inputs(name))
    ref = golden_digests(name)
    return all(str(mine[k]) == str(ref[k]) for k in ref)


def golden_rows(name: str):
    """Point subset at which a large fixture stores its per-point outputs
    (c2n4 / c2n8: every 3rd / 8th point), else all points."""
    z = golden(name)
    return z["rows"] if "rows" in z else slice(None)


def golden_weights(name: str):
    """ifgf_apply input of a fixture: stored, or phi * weights rebuilt from y
    (reference operators.py:336; c2n4 / c2n8 do not store it)."""
    z = golden(name)
    if "weights" in z:
        return z["weights"]
    from paper_2408_02274_b200.operator import DensityBlock
    disc = inputs(name)["disc"]
    n = disc.n_points
    y = z["y"]
    t1, t2 = disc.tangent1, disc.tangent2
    m = y[0:n, None] * t1 + y[n:2 * n, None] * t2
    j = y[2 * n:3 * n, None] * t1 + y[3 * n:, None] * t2
    return DensityBlock.from_currents(disc, j, m).values * disc.weights
