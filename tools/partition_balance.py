#!/usr/bin/env python
"""Load balance of the multi-GPU partition (DESIGN 7), measured on ONE GPU:
for P logical ranks, each rank's plan (its Morton range of level-3 subtrees
and its patch range) is built and its far phase and near phase are timed
with CUDA events, one rank after another (no collective, nothing waits on
another rank).  Reports per-rank times, max/mean imbalance and the bytes
each NCCL all-reduce moves per matvec.  This is a projection input, not a
multi-GPU measurement: the pool grants one GPU per call.

  python tools/partition_balance.py --n-refine 8 --ranks 1 2 4 8
"""

from __future__ import annotations

import argparse
import gc
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


class _NoComm:
    def all_reduce(self, t, group=None):
        pass


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-refine", type=int, default=8)
    ap.add_argument("--k0-pi", type=float, default=None)
    ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()

    import numpy as np
    import torch
    import bench
    from paper_2408_02274_b200 import _lib
    from paper_2408_02274_b200.build import build
    from paper_2408_02274_b200.engine import device_stream
    from paper_2408_02274_b200.operator import MullerOperator
    from paper_2408_02274_b200.partition import DistributedMullerOperator, level3_partition

    build()
    torch.cuda.set_device(0)
    disc, mats, y_np, name = bench.workload(args.n_refine, args.k0_pi)
    tree, hier, smap, mom, cp = bench.plan_inputs(disc, mats)
    lib, st = _lib.load(), device_stream()
    y = torch.from_numpy(y_np).cuda()
    n = disc.n_points
    rows = []
    for P in args.ranks:
        parts = level3_partition(tree, hier, P, disc.n_patches, disc.n_c)
        far_ms, near_ms = [], []
        for part in parts:
            op = MullerOperator(disc, mats, smap, mom, (cp.ell_idx, cp.src_idx),
                                tree=tree, hierarchy=hier, stream_parts=1)
            dop = DistributedMullerOperator(op, part)
            dop.dist = _NoComm()
            out = torch.zeros_like(y)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            best_f, best_n = 1e30, 1e30
            for r in range(args.reps + 1):
                torch.cuda.synchronize()
                ev[0].record(torch.cuda.current_stream())
                _lib.check(lib.ifgfb_muller_far_phase(op.plan.handle, y.data_ptr(), st), "far")
                ev[1].record(torch.cuda.current_stream())
                _lib.check(lib.ifgfb_muller_near_phase(op.plan.handle, y.data_ptr(),
                                                       out.data_ptr(), st), "near")
                ev[2].record(torch.cuda.current_stream())
                torch.cuda.synchronize()
                if r:
                    best_f = min(best_f, ev[0].elapsed_time(ev[1]))
                    best_n = min(best_n, ev[1].elapsed_time(ev[2]))
            far_ms.append(best_f)
            near_ms.append(best_n)
            del dop, op
            gc.collect()
            torch.cuda.empty_cache()
        tot = [f + m for f, m in zip(far_ms, near_ms)]
        rows.append({"ranks": P, "far_ms": [round(v, 3) for v in far_ms],
                     "near_ms": [round(v, 3) for v in near_ms],
                     "max_rank_ms": round(max(tot), 3), "mean_rank_ms": round(float(np.mean(tot)), 3),
                     "imbalance_max_over_mean": round(max(tot) / float(np.mean(tot)), 3),
                     "allreduce_bytes": {"far_partials": 2 * 16 * n * 16, "result_rows": 4 * n * 16}})
        print(json.dumps(rows[-1]), flush=True)
    base = rows[0]["max_rank_ms"] if rows and rows[0]["ranks"] == 1 else None
    print(json.dumps({"workload": name, "unknowns": 4 * n,
                      "projected_speedup_compute_only": {
                          r["ranks"]: (round(base / r["max_rank_ms"], 2) if base else None)
                          for r in rows}}), flush=True)


if __name__ == "__main__":
    main()
