"""Quick GPU check of the full N-Muller apply against golden reference outputs."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2408_02274_b200 import surface  # noqa: E402
from paper_2408_02274_b200.operator import (DensityBlock, MaterialPair,  # noqa: E402
                                            build_muller_operator)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


for name in sys.argv[1:] or ["s1", "c1"]:
    z = np.load(f"tests/golden/{name}.npz")
    nr, nc, k0pi, eps = z["config"]
    disc = surface.make_sphere_surface(int(nr), int(nc))
    k0 = k0pi * np.pi
    mats = MaterialPair(1.0, 1.0, eps, 1.0, k0)
    t0 = time.time()
    op = build_muller_operator(disc, mats)
    t1 = time.time()
    y = z["y"]
    out = op.apply(y)
    t2 = time.time()
    m, j = op.decode(y)
    dens = DensityBlock.from_currents(disc, j, m)
    s_val, d_val = op.potentials(dens)
    def rel_rows(a, key):   # the larger goldens keep a row subset of the potentials
        ref = z[key]
        if a.shape != ref.shape and "rows" in z.files:
            a = a[..., z["rows"]]
        return f"{rel(a, ref):.3e}" if a.shape == ref.shape else "n/a"
    print(f"{name}: N={disc.n_points} build {t1 - t0:.2f}s apply(first) {t2 - t1:.3f}s | "
          f"apply rel {rel(out, z['apply_y']):.3e} S rel {rel_rows(s_val, 's_val')} "
          f"D rel {rel_rows(d_val, 'd_val')} (ref floor lin {float(z['floor_linearity']):.2e})")
    dev = torch.device("cuda")
    yd = torch.from_numpy(y).to(dev)
    od = torch.empty_like(yd)
    for _ in range(3):
        op.apply_device(yd, od)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        op.apply_device(yd, od)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"   device apply {ms:.3f} ms -> {4 * disc.n_points / (ms * 1e-3):.3e} unknowns*matvec/s, "
          f"launches {op.last_launches()}, near {op.near_stats}")
    t0 = time.time()
    for _ in range(reps):
        op.apply(y)
    t1 = time.time()
    print(f"   host apply (e2e) {(t1 - t0) / reps * 1e3:.3f} ms")
