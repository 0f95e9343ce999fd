#!/usr/bin/env python
"""Per-rank work and memory of the multi-GPU matvec (DESIGN 7), measured on
ONE GPU: for P logical ranks, each rank's own plan (its window of level-3
subtrees and its target rows, built from the tree-only partition exactly as
a rank process builds it) is created, its far phase and near phase are
timed with CUDA events, and it is freed before the next rank (one rank at a
time: no collective, nothing waits on another rank).  Reports per-rank
times, plan build times, device bytes, max/mean imbalance and the bytes each
collective moves per matvec.  A projection input, not a multi-GPU
measurement: the pool grants one GPU per call.

  python tools/partition_balance.py --n-refine 8 --ranks 1 2 4 8
"""

from __future__ import annotations

import argparse
import gc
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-refine", type=int, default=8)
    ap.add_argument("--k0-pi", type=float, default=None)
    ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--moments", choices=["host", "device"], default="device")
    args = ap.parse_args()

    import torch
    import bench
    from paper_2408_02274_b200 import octree
    from paper_2408_02274_b200.build import build
    from paper_2408_02274_b200.partition import DistributedMullerOperator, level3_partition

    build()
    torch.cuda.set_device(0)
    disc, mats, y_np, name = bench.workload(args.n_refine, args.k0_pi)
    kmax = max(abs(mats.kappa_e), abs(mats.kappa_i))
    tree = octree.build_box_tree(disc.points, kmax)
    y = torch.from_numpy(y_np).cuda()
    rows = []
    for P in args.ranks:
        parts = level3_partition(tree, None, P, disc.n_patches, disc.n_c)
        res = []
        for part in parts:
            t0 = time.time()
            op = DistributedMullerOperator(disc, mats, part, tree=tree, exchange=False,
                                           device_moments=args.moments == "device")
            t_plan = time.time() - t0
            far, near = [], []
            for _ in range(args.reps + 1):
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                e[0].record()
                op.far_phase(y)
                e[1].record()
                c = op.xfar_mine.numel()
                op.xfar_mine.copy_(op.xfar[part.rank * c:(part.rank + 1) * c])
                op.near_phase(y)
                e[2].record()
                torch.cuda.synchronize()
                far.append(e[0].elapsed_time(e[1]))
                near.append(e[1].elapsed_time(e[2]))
            res.append({"rank": part.rank, "box3": part.box3, "targets": part.targets,
                        "far_ms": min(far[1:]), "near_ms": min(near[1:]),
                        "plan_s": round(t_plan, 1),
                        "device_gib": round(op.device_bytes() / 2**30, 3),
                        "modelled_work": part.work})
            del op
            gc.collect()
            torch.cuda.empty_cache()
        tot = [r["far_ms"] + r["near_ms"] for r in res]
        chunk = parts[0].chunk
        row = {"workload": name, "ranks": P, "per_rank": res,
               "max_ms": max(tot), "mean_ms": sum(tot) / P,
               "imbalance": max(tot) / (sum(tot) / P),
               "reduce_scatter_mb": P * chunk * 32 * 16 / 1e6,
               "all_gather_mb": P * chunk * 4 * 16 / 1e6}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if rows and rows[0]["ranks"] == 1:
        t1 = rows[0]["max_ms"]
        for r in rows:
            print(f"P={r['ranks']}: slowest rank {r['max_ms']:.2f} ms, imbalance "
                  f"{r['imbalance']:.3f}, projected compute speedup {t1 / r['max_ms']:.2f}x, "
                  f"max device {max(x['device_gib'] for x in r['per_rank']):.2f} GiB",
                  flush=True)


if __name__ == "__main__":
    main()
