"""Diagnostic: D_far = (S(x + h n) - S(x)) / h from the GPU far field against
direct sums at the rows where D is largest (sphere(n, 10))."""
import gc
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import bench
from paper_2408_02274_b200.engine import ifgf_apply
from paper_2408_02274_b200.operator import DensityBlock, MullerOperator

n, k0pi = int(sys.argv[1]), (float(sys.argv[2]) if sys.argv[2] != "-" else None)
geometry = sys.argv[3] if len(sys.argv) > 3 else "sphere"
disc, mats, y, name = bench.workload(n, k0pi, geometry)
tree, hier, smap, mom, cp = bench.plan_inputs(disc, mats)
N = disc.n_points
nrm = disc.normals
rng = np.random.default_rng(3)
m = np.cross(nrm, rng.normal(size=3) + 1j * rng.normal(size=3))
j = np.cross(nrm, rng.normal(size=3) + 1j * rng.normal(size=3))
dens = DensityBlock.from_currents(disc, j, m)
w = dens.values * disc.weights
far, far_d = ifgf_apply(tree, hier, w, mats.kappas, displaced_normals=nrm, displaced_step=1e-6)
dfar = (far_d - far) / 1e-6
hier.__dict__.pop("_b200_plans", None); gc.collect()
op = MullerOperator(disc, mats, smap, mom, (cp.ell_idx, cp.src_idx), tree=tree, hierarchy=hier)
s, d = op.potentials(dens)
print(name, "stream parts", getattr(op.plan, "stream_parts", None))
q = lambda a: np.percentile(np.abs(a), [50, 99, 99.9, 100])
print("D p50/p99/p99.9/max", q(d), " dfar", q(dfar[:6]), " S", q(s))
out = op.apply(y)
print("apply p50/p99/p99.9/max", q(out))
blk = np.abs(out).reshape(4, N).max(0)
print("top apply rows", [(disc.decode_index(int(e)), float(blk[e])) for e in np.argsort(-blk)[:6]])
rows = np.argsort(-np.abs(d).max(axis=(0, 1)))[:6]
dd = tree.depth
coords = tree.level(dd).coords[tree.point_boxes(dd)]
wt = w[:, tree.perm]
for ell in rows:
    t = tree.iperm[ell]
    far_m = np.abs(coords - coords[t]).max(axis=1) >= 2
    x = tree.points[t]; nx = nrm[ell]
    r0 = np.linalg.norm(x - tree.points[far_m], axis=1)
    r1 = np.linalg.norm(x + 1e-6 * nx - tree.points[far_m], axis=1)
    out = []
    for k, kap in enumerate(mats.kappas):
        g0 = np.exp(1j * kap * r0) / (4 * np.pi * r0)
        g1 = np.exp(1j * kap * r1) / (4 * np.pi * r1)
        out.append(((g1 - g0) / 1e-6 * wt[:6, far_m]).sum(1))
    naive = np.stack(out, 1)
    print(disc.decode_index(int(ell)), "|D| max %.3g" % np.abs(d[:, :, ell]).max(),
          "|dfar gpu| %.3g" % np.abs(dfar[:6, :, ell]).max(), "|dfar naive| %.3g" % np.abs(naive).max(),
          "|S| %.3g" % np.abs(s[:, :, ell]).max(), "singular patches", list(smap.singular_patches(ell)),
          "min src dist %.3g" % r0.min())
