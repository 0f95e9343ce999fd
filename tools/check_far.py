"""Quick GPU check of the far field against the golden reference outputs."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2408_02274_b200 import octree, surface  # noqa: E402
from paper_2408_02274_b200.engine import FarFieldPlan, ifgf_apply  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


for name in sys.argv[1:] or ["rand", "s1", "c1"]:
    if name == "rand":
        z = np.load("tests/golden/rand_ifgf.npz")
        disc = surface.make_sphere_surface(1, 6)
        kap = tuple(z["kappas"])
        w = z["weights"]
    else:
        z = np.load(f"tests/golden/{name}.npz")
        nr, nc, k0pi, eps = z["config"]
        disc = surface.make_sphere_surface(int(nr), int(nc))
        k0 = k0pi * np.pi
        kap = (k0, k0 * np.sqrt(eps))
        w = z["weights"]
    t0 = time.time()
    tree = octree.build_box_tree(disc.points, max(abs(k) for k in kap))
    hier = octree.build_cone_hierarchy(tree)
    t1 = time.time()
    out, od = ifgf_apply(tree, hier, w, kap, displaced_normals=disc.normals,
                         displaced_step=1e-6)
    torch.cuda.synchronize()
    t2 = time.time()
    out, od = ifgf_apply(tree, hier, w, kap, displaced_normals=disc.normals,
                         displaced_step=1e-6)
    t3 = time.time()
    ref, refd = z["far"], z["far_disp"]
    dg = (od - out) / 1e-6
    dr = (refd - ref) / 1e-6
    print(f"{name}: N={disc.n_points} plan {t1 - t0:.2f}s first {t2 - t1:.2f}s "
          f"second {t3 - t2:.3f}s | far rel {rel(out, ref):.3e} disp rel "
          f"{rel(od, refd):.3e} D_far rel {rel(dg, dr):.3e}")
    # timing of the device apply alone
    plan = list(hier._b200_plans.values())[0][0]
    dev = torch.device("cuda")
    wd = torch.from_numpy(np.ascontiguousarray(w)).to(dev)
    o = torch.empty((w.shape[0], len(kap), disc.n_points), dtype=torch.complex128, device=dev)
    o2 = torch.empty_like(o)
    for _ in range(3):
        plan.far_apply_device(wd, kap, o, o2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 10
    for _ in range(reps):
        plan.far_apply_device(wd, kap, o, o2)
    e1.record()
    torch.cuda.synchronize()
    print(f"   device far_apply {e0.elapsed_time(e1) / reps:.3f} ms, launches {plan.last_launches()}, "
          f"plan bytes {plan.device_bytes() / 1e6:.1f} MB, stats {plan.stats}")
