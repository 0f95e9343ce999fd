"""Small driver for ncu: build the bench operator and run a few applies."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2408_02274_b200.operator import MullerOperator  # noqa: E402

n_refine = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
disc, mats, y, name = bench.workload(n_refine)
tree, hier, smap, mom, cp = bench.plan_inputs(disc, mats)
op = MullerOperator(disc, mats, smap, mom, (cp.ell_idx, cp.src_idx), tree=tree, hierarchy=hier)
yd = torch.from_numpy(y).cuda()
out = torch.empty_like(yd)
for _ in range(reps):
    op.apply_device(yd, out)
torch.cuda.synchronize()
print("done", name, float(out.abs().sum()))
