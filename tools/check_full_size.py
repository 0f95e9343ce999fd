"""Size-independent checks of the far field at a full BASELINE size on the
GPU (default: cfg 5, sphere(45,10), k0 = 32 pi, 1.2 M points, streaming and
on-device geometry active): accuracy against direct sums at sampled targets
(the reference's own bar, tests/test_ifgf.py:296-308: 1.5e-4 at its sizes),
the displaced outputs against direct sums at x + h n, linearity and bitwise
run-to-run determinism.

  python tools/check_full_size.py [--n-refine 45 --k0-pi 32 --targets 64]

Prints one JSON line (kept under profiles/).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def naive_far_at(tree, w, kappas, targets, disp=None):
    """Direct far sums (reference naive_far_sums, tests/test_ifgf.py:22-38) at
    a few targets (original indices): sources outside the target's
    finest-level neighbour boxes; disp: evaluate at x + disp[ell]."""
    d = tree.depth
    coords = tree.level(d).coords[tree.point_boxes(d)]
    wt = np.atleast_2d(w)[:, tree.perm]
    out = np.zeros((wt.shape[0], len(kappas), len(targets)), dtype=complex)
    for j, ell in enumerate(targets):
        t = tree.iperm[ell]
        far = np.abs(coords - coords[t]).max(axis=1) >= 2
        x = tree.points[t] if disp is None else tree.points[t] + disp[ell]
        r = np.linalg.norm(x - tree.points[far], axis=1)
        for k, kap in enumerate(kappas):
            out[:, k, j] = (np.exp(1j * kap * r) / (4 * np.pi * r) * wt[:, far]).sum(1)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-refine", type=int, default=45)
    ap.add_argument("--k0-pi", type=float, default=32)
    ap.add_argument("--targets", type=int, default=64)
    args = ap.parse_args()
    import torch
    import bench
    from paper_2408_02274_b200 import octree
    from paper_2408_02274_b200.build import build
    from paper_2408_02274_b200.engine import FarFieldPlan, k4_mode
    build()
    disc, mats, _, name = bench.workload(args.n_refine, args.k0_pi, "sphere")
    kap = tuple(float(abs(k)) for k in mats.kappas)
    t0 = time.time()
    tree = octree.build_box_tree(disc.points, max(kap))
    hier = octree.build_cone_hierarchy(tree, device=disc.n_points > 100_000)
    step = 1e-6
    plan = FarFieldPlan(tree, hier, disc.normals, step, kappas=kap)
    parts = plan.auto_stream()
    t_plan = time.time() - t0
    n = disc.n_points
    rng = np.random.default_rng(7)
    w = rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n))
    w2 = rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n))
    dev = torch.device("cuda")

    def run(wh):
        wd = torch.from_numpy(np.ascontiguousarray(wh)).to(dev)
        o = torch.empty((wh.shape[0], len(kap), n), dtype=torch.complex128, device=dev)
        od = torch.empty_like(o)
        plan.far_apply_device(wd, kap, o, od)
        return o.cpu().numpy(), od.cpu().numpy()

    a, ad = run(w)
    a2, ad2 = run(w)
    b, _ = run(w2)
    c, _ = run(w + 0.5j * w2)
    idx = rng.choice(n, args.targets, replace=False)
    rel = lambda x, y: float(np.linalg.norm(x - y) / np.linalg.norm(y))
    ref = naive_far_at(tree, w, kap, idx)
    refd = naive_far_at(tree, w, kap, idx, disp=step * disc.normals)
    line = {
        "workload": name, "points": int(n), "depth": int(tree.depth),
        "k4_kernel": k4_mode(), "stream_parts": int(parts),
        "geometry_on_device_levels": sorted(plan.otf_levels),
        "far_plan_build_s": round(t_plan, 1), "targets": int(args.targets),
        "far_vs_direct_sums_rel_l2": rel(a[:, :, idx], ref),
        "far_displaced_vs_direct_sums_rel_l2": rel(ad[:, :, idx], refd),
        "dfar_vs_direct_rel_l2": rel((ad - a)[:, :, idx] / step, (refd - ref) / step),
        "linearity_max_rel": float(np.abs(c - a - 0.5j * b).max() / np.abs(c).max()),
        "bitwise_run_to_run": bool(np.array_equal(a, a2) and np.array_equal(ad, ad2)),
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
