"""Plan-build time and host memory per stage (no device work beyond the
plan upload): python tools/plan_memory.py n_refine"""
import resource
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2408_02274_b200 import nearfield, octree  # noqa: E402

T0 = time.time()


def cur():
    return int(open("/proc/self/statm").read().split()[1]) * 4096 / 1e9


def peak():
    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6


def mark(what, t):
    print(f"{what:28s} {time.time() - t:8.1f}s  rss {cur():7.2f} GB  peak {peak():7.2f} GB"
          f"  (t={time.time() - T0:.0f}s)", flush=True)


n = int(sys.argv[1])
disc, mats, y, name = bench.workload(n)
print(name, "points", disc.n_points, flush=True)
kmax = max(abs(mats.kappa_e), abs(mats.kappa_i))
t = time.time(); tree = octree.build_box_tree(disc.points, kmax); mark("tree", t)
t = time.time(); hier = octree.build_cone_hierarchy(tree); mark("cone hierarchy", t)
t = time.time(); smap = nearfield.classify_targets(disc); mark("classify", t)
t = time.time()
mom = nearfield.compute_moments(disc, smap, nearfield.SingularQuadratureConfig(), mats.kappas)
mark("moments", t)
t = time.time(); cp = nearfield.correction_pairs(disc, tree, smap); mark("corrections", t)
dev = 0
for d in range(4, tree.depth + 1):
    t = time.time(); ap = octree.accumulation_plan(tree, hier, d)
    mark(f"accum plan {d} ({ap.n_types} types)", t)
    ng = int(ap.inst_crow_off[-1])
    est = ap.n_types * 75 * 72 + ap.n_instances * (12 * 16 + 4 * 4) + ng * 4 + \
        hier.level(d - 1).n_segments * (75 + 6)
    dev += est
    print(f"   level {d}: types {ap.n_types} instances {ap.n_instances} groups {ng}"
          f" types/inst {ap.n_types / max(1, ap.n_instances):.2f}  device est {est / 1e9:.1f} GB",
          flush=True)
pairs = [hier.level(d).cpt_idx.size for d in range(3, tree.depth + 1)]
print(f"emission pairs per level {pairs}; device est {sum(pairs) * 72 / 1e9:.1f} GB + partial "
      f"{max(pairs) * 512 / 1e9:.1f} GB; segments {[hier.level(d).n_segments for d in range(3, tree.depth + 1)]}")
print(f"propagation device estimate {dev / 1e9:.1f} GB", flush=True)
if "--op" in sys.argv:
    from paper_2408_02274_b200.operator import MullerOperator
    t = time.time()
    op = MullerOperator(disc, mats, smap, mom, (cp.ell_idx, cp.src_idx), tree=tree,
                        hierarchy=hier)
    mark("MullerOperator (upload)", t)
