"""How much K4 (propagation) gains from processing G parent rows of one box
per CTA: MMA row tiles per instance and distinct child blocks per instance
for several groupings of a level's parent rows (host analysis, no GPU).

  python tools/group_analysis.py --n-refine 4 --k0-pi 4

Groupings: single rows (today's kernel), consecutive row pairs / quads of
one box with equal (i_s, i_t>>1, i_p>>1) ("quad"), and whole radial columns.
For each: tiles per (row, child) instance if the tiles of one sigma group
are formed over all the group's nodes in the CTA (8 rows per tile), the
ideal 75/8, and the number of 19 KB child blocks fetched per instance.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-refine", type=int, default=4)
    ap.add_argument("--k0-pi", type=float, default=4)
    args = ap.parse_args()
    from paper_2408_02274_b200 import octree, surface
    disc = surface.make_sphere_surface(args.n_refine, 10)
    tree = octree.build_box_tree(disc.points, args.k0_pi * np.pi * 1.5)
    hier = octree.build_cone_hierarchy(tree)
    for d in range(tree.depth, 3, -1):
        acc = octree.accumulation_plan(tree, hier, d, device=False)
        pcl = hier.level(d - 1)
        n_rows = acc.inst_off.size - 1
        ni = np.diff(acc.inst_off)
        rows = np.nonzero(ni > 0)[0]
        seg = pcl.seg_ids[rows]
        box = np.searchsorted(pcl.seg_off, rows, side="right") - 1
        two_na = 2 * pcl.n_a
        i_p = seg % two_na
        i_t = (seg // two_na) % pcl.n_a
        i_s = seg // (two_na * pcl.n_a)
        # global sigma (child row) per (instance, node)
        def inst_node_crow(r):
            out = []
            for i in range(acc.inst_off[r], acc.inst_off[r + 1]):
                t = acc.inst_type[i]
                out.append(acc.crow[acc.inst_crow_off[i] + acc.gid[t].astype(np.int64)])
            return out      # list over children (same order for rows of a box)

        def measure(keys, name):
            # group rows by key; per group and child: tiles = sum ceil(n_g / 8)
            order = np.argsort(keys, kind="stable")
            ks = keys[order]
            cut = np.nonzero(np.diff(ks))[0] + 1
            groups = np.split(order, cut)
            rng = np.random.default_rng(0)
            pick = rng.choice(len(groups), size=min(len(groups), 1500), replace=False)
            tiles = blocks = insts = 0
            sizes = []
            for gi in pick:
                g = groups[gi]
                sizes.append(g.size)
                per_child = [inst_node_crow(rows[r]) for r in g]
                nch = len(per_child[0])
                for c in range(nch):
                    cr = np.concatenate([pc[c] for pc in per_child])
                    _, cnt = np.unique(cr, return_counts=True)
                    tiles += int(np.sum((cnt + 7) // 8))
                    blocks += cnt.size
                    insts += g.size
            print(f"  {name:28s} rows/CTA {np.mean(sizes):5.2f}  tiles/inst {tiles / insts:6.2f} "
                  f"(fill {75 / 8 / (tiles / insts):.3f})  blocks/inst {blocks / insts:6.2f}")

        print(f"level {d}->{d-1}: {rows.size} rows, {acc.n_instances} instances, "
              f"n_s {pcl.n_s} n_a {pcl.n_a}")
        base = box.astype(np.int64) * (1 << 40)
        measure(base + seg, "single row")
        measure(base + ((i_s * pcl.n_a + i_t) * two_na + (i_p >> 1)) , "phi pair")
        measure(base + ((i_s * pcl.n_a + (i_t >> 1)) * two_na + (i_p >> 1)), "theta x phi quad")
        measure(base + (((i_s >> 1) * pcl.n_a + (i_t >> 1)) * two_na + (i_p >> 1)), "s x theta x phi oct")
        measure(base + (i_t >> 1) * two_na + (i_p >> 1), "quad x all s")


if __name__ == "__main__":
    main()
