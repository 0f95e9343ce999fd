"""Stage timings and host peak RSS of the plan build for one bench workload.

  IFGFB_PLAN_LOG=1 python tools/plan_profile.py --n-refine 45 --k0-pi 32

Prints the host (cores, RAM), every plan stage (tree, cones, classify,
moments, corrections, near-field description, per-level accumulation plan /
row tiles / upload, emission) and the peak RSS.  Used to decide which plan
stages to move to native code.
"""

from __future__ import annotations

import argparse
import os
import resource
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("IFGFB_PLAN_LOG", "1")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-refine", type=int, default=45)
    ap.add_argument("--k0-pi", type=float, default=32)
    ap.add_argument("--geometry", default="sphere")
    ap.add_argument("--host-moments", action="store_true")
    args = ap.parse_args()
    import bench
    from paper_2408_02274_b200 import nearfield
    from paper_2408_02274_b200.build import build
    from paper_2408_02274_b200.operator import MullerOperator
    build()
    print(f"host: {os.cpu_count()} cpus, "
          f"{os.sysconf('SC_PAGE_SIZE') * os.sysconf('SC_PHYS_PAGES') / 2**30:.0f} GiB RAM",
          file=sys.stderr, flush=True)
    disc, mats, y, name = bench.workload(args.n_refine, args.k0_pi, args.geometry)
    print(name, disc.n_points, file=sys.stderr, flush=True)
    t0 = time.time()
    tree, hier, smap, mom, cp = bench.plan_inputs(disc, mats, not args.host_moments)
    print(f"[plan] corrections {time.time() - t0:.1f}s nnz={cp.nnz}", file=sys.stderr,
          flush=True)
    op = MullerOperator(disc, mats, smap, mom, (cp.ell_idx, cp.src_idx),
                        tree=tree, hierarchy=hier)
    print(f"[plan] total {time.time() - t0:.1f}s stream_parts={op.plan.stream_parts} "
          f"otf={sorted(op.plan.otf_levels)} device_bytes={op.plan.device_bytes() / 2**30:.1f} GiB",
          file=sys.stderr, flush=True)
    rss = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20
    print(f"[plan] peak RSS {rss:.1f} GiB", file=sys.stderr, flush=True)
    _ = nearfield


if __name__ == "__main__":
    main()
