"""Diagnostic: magnitudes of the far field, potentials and apply rows for a
sphere(n, 10) configuration (locates rows that blow up)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import bench
from paper_2408_02274_b200.engine import ifgf_apply
from paper_2408_02274_b200.operator import DensityBlock, MullerOperator
from test_gpu_far import _naive_far_at

n, k0pi = int(sys.argv[1]), float(sys.argv[2])
disc, mats, y, name = bench.workload(n, k0pi)
tree, hier, smap, mom, cp = bench.plan_inputs(disc, mats)
rng = np.random.default_rng(3)
N = disc.n_points
w = rng.normal(size=(2, N)) + 1j * rng.normal(size=(2, N))
far, _ = ifgf_apply(tree, hier, w, mats.kappas)
idx = rng.choice(N, 60, replace=False)
ref = _naive_far_at(tree, w, mats.kappas, idx)
print(name, "depth", tree.depth, "far vs naive rel", np.linalg.norm(far[:, :, idx] - ref) / np.linalg.norm(ref))
q = lambda a: np.percentile(np.abs(a), [50, 99, 100])
print("far |.| p50/p99/max", q(far))
hier.__dict__.pop("_b200_plans", None)
import gc; gc.collect()
op = MullerOperator(disc, mats, smap, mom, (cp.ell_idx, cp.src_idx), tree=tree, hierarchy=hier)
print("stream parts", getattr(op.plan, "stream_parts", None), "otf", sorted(op.plan.otf_levels),
      "plan GB", op.plan.device_bytes() / 1e9, "free GB", torch.cuda.mem_get_info()[0] / 1e9)
m, j = op.decode(y)
nrm = disc.normals
m = m - (m * nrm).sum(1)[:, None] * nrm
j = j - (j * nrm).sum(1)[:, None] * nrm
dens = DensityBlock.from_currents(disc, j, m)
s, d = op.potentials(dens)
print("S p50/p99/max", q(s), "D", q(d))
big = np.argsort(-np.abs(s).max(axis=(0, 1)))[:5]
print("largest S rows (patch, i, j):", [disc.decode_index(int(e)) for e in big], np.abs(s).max(axis=(0, 1))[big])
out = op.apply(y)
print("apply |.| p50/p99/max", q(out), " |y| max", np.abs(y).max())
blk = np.abs(out).reshape(4, N)
big = np.argsort(-blk.max(0))[:8]
print("largest apply rows:", [(disc.decode_index(int(e)), float(blk[:, e].max())) for e in big])
print("moments |beta| max", np.abs(mom.csr_blocks).max() if getattr(mom, "csr_blocks", None) is not None else
      max(np.abs(g.beta_s).max() for g in mom.groups.values()),
      "n singular pairs", smap.patch_ids.size, "per target max", np.diff(smap.offsets).max())
