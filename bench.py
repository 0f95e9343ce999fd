#!/usr/bin/env python
"""Benchmark: IFGF-accelerated N-Muller matvec throughput on B200.

metric  = unknowns * matvec / s  (4N unknowns per apply, BASELINE.json)
value   = device throughput with y resident in HBM (CUDA events, L2 flushed
          between steps)
e2e     = same metric through the public host API (MullerOperator.apply on a
          numpy vector: pinned staging, H2D, apply, D2H inside the timed call)

Workload (BASELINE.json configs[1], cfg-2 family): unit dielectric sphere,
eps_r = 2.25, 6 x n^2 patches on 10x10 Chebyshev grids, k0 = pi * n (fixed
points per wavelength, reference cli.py:300-307), y ~ N(0,1) + i N(0,1)
(seed 0), reference default IFGF parameters.  Default n = 4 (38,400
unknowns).

--impl reference: the reference algorithm's CPU implementation (the numpy
oracle restatement, `oracle/`, since the reference is Python and cannot be
compiled) on this host's cores, on a bounded sample of the same workload.

Multi-GPU (torchrun, N > 1): ONE matvec partitioned over the ranks
(paper_2408_02274_b200/partition.py): Morton ranges of level-3 subtrees for
the upward pass, patch ranges for near field and assembly, NCCL all-reduce
of the far-field partials and of the result rows (strong scaling); the
timed region is barrier-bracketed and the max over ranks is reported.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FP64_PEAK_TFLOPS = 37.0   # DMMA m8n8k4 f64, measured (profiles/fp64_peak_r01.txt)
W_PROP = 75 * 75 * 16 * 4          # FLOP per (parent segment, child) instance
W_COEF = 16 * (3 * 3 * 25 + 5 * 5 * 15 + 5 * 5 * 15) * 4   # K3 per segment
W_EMIT = 2 * 75 * 16 * 4           # per (box, target) pair, x and x + h n
W_LEAF = 128                       # per (node, source) pair (2 kernels x 8 ch)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--n-refine", type=int, default=4)
    ap.add_argument("--k0-pi", type=float, default=None,
                    help="k0 / pi (default n_refine: ~10 points per wavelength; cfg 5 is 45 / 32)")
    ap.add_argument("--geometry", choices=["sphere", "superellipsoid", "slab"],
                    default="sphere", help="BASELINE cfg 1/2/5, cfg 3, cfg 4 bodies")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--device-moments", action="store_true",
                    help="singular moments from the plan-time GPU kernel (large surfaces)")
    ap.add_argument("--no-gmres", action="store_true")
    ap.add_argument("--max-rss-gb", type=float, default=0.0,
                    help="abort (kill this process) if host RSS exceeds this")
    ap.add_argument("--force-partition", action="store_true",
                    help="use the partitioned (multi-GPU) operator even at N=1")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload(n_refine, k0_pi=None, geometry="sphere"):
    """BASELINE configs: 'sphere' = cfg 1/2/5 family (sphere(n, 10), k0 = pi n
    by default, eps_r 2.25); 'superellipsoid' = cfg 3 (|x/2|^4 + |y|^4 +
    |z/0.5|^4 = 1, n x n subpatches per face on 12 x 12 grids, eps_r 4,
    2a = 8 wavelengths -> k0 = 4 pi); 'slab' = cfg 4 (exponent-8
    superellipsoid with half-extents 20 x 0.25 x 0.11 wavelengths, eps_r
    12.11, (16n, 2n, n) aspect-graded splits on 10 x 10 grids, wavelength 1
    -> k0 = 2 pi)."""
    import numpy as np
    from paper_2408_02274_b200 import surface
    from paper_2408_02274_b200.operator import MaterialPair
    if geometry == "sphere":
        disc = surface.make_sphere_surface(n_refine, 10)
        k0_pi = n_refine if k0_pi is None else k0_pi
        eps = 2.25
        name = f"sphere(n_refine={n_refine}, n_c=10) k0={k0_pi:g}pi eps_r=2.25"
    elif geometry == "superellipsoid":
        disc = surface.make_superellipsoid_surface(n_refine, 12, (2.0, 1.0, 0.5), 4.0)
        k0_pi = 4.0 if k0_pi is None else k0_pi
        eps = 4.0
        name = (f"superellipsoid(|x/2|^4+|y|^4+|z/0.5|^4=1, {n_refine}x{n_refine} "
                f"subpatches/face, n_c=12) k0={k0_pi:g}pi eps_r=4")
    elif geometry == "slab":
        k0_pi = 2.0 if k0_pi is None else k0_pi
        lam = 2.0 / k0_pi
        splits = (16 * n_refine, 2 * n_refine, n_refine)
        disc = surface.make_superellipsoid_surface(
            splits, 10, (20.0 * lam, 0.25 * lam, 0.11 * lam), 8.0)
        eps = 12.11
        name = (f"slab(superellipsoid p=8, 20 x 0.25 x 0.11 wavelengths, splits "
                f"{splits}, n_c=10) k0={k0_pi:g}pi eps_r=12.11")
    else:
        raise ValueError(f"unknown geometry {geometry}")
    mats = MaterialPair(1.0, 1.0, eps, 1.0, np.pi * k0_pi)
    n = disc.n_points
    rng = np.random.default_rng(0)
    y = rng.normal(size=4 * n) + 1j * rng.normal(size=4 * n)
    return disc, mats, y, name


def plan_inputs(disc, mats, device_moments=False):
    from paper_2408_02274_b200 import nearfield, octree
    kmax = max(abs(mats.kappa_e), abs(mats.kappa_i))
    t0 = time.time()
    stage = lambda what: print(f"[plan] {what} {time.time() - t0:.1f}s", file=sys.stderr,
                               flush=True)
    tree = octree.build_box_tree(disc.points, kmax)
    stage("tree")
    hier = octree.build_cone_hierarchy(tree)
    stage("cones")
    smap = nearfield.classify_targets(disc)
    stage("classify")
    cfg = nearfield.SingularQuadratureConfig()
    if device_moments:
        mom = nearfield.compute_moments_device(disc, smap, cfg, mats.kappas, groups=False)
    else:
        mom = nearfield.compute_moments(disc, smap, cfg, mats.kappas)
    stage("moments")
    cp = nearfield.correction_pairs(disc, tree, smap)
    return tree, hier, smap, mom, cp


def work_counts(tree, hier):
    """Algorithmic FLOP per matvec from the plan."""
    from paper_2408_02274_b200 import octree
    D = tree.depth
    prop = {}
    for d in range(4, D + 1):
        ap = octree.accumulation_plan(tree, hier, d, geometry=False)
        prop[d] = W_PROP * ap.n_instances + W_COEF * hier.level(d - 1).n_segments
    cl, lvl = hier.level(D), tree.level(D)
    leaf = W_LEAF * 75 * int((cl.seg_off[1:] - cl.seg_off[:-1]) @ lvl.pt_count)
    emit = W_EMIT * sum(hier.level(d).cpt_idx.size for d in range(3, D + 1))
    return {"prop_by_level": prop, "prop": sum(prop.values()), "leaf": leaf,
            "leaf_coef": W_COEF * cl.n_segments, "emit": emit,
            "total": sum(prop.values()) + leaf + W_COEF * cl.n_segments + emit}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = ROOT / "gpurun_out" / f"clocks_{index}_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.path.parent.mkdir(exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in self.path.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 8:
                rows.append(parts)
        try:
            self.path.unlink()
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def cpu_baseline(disc, mats, y, inputs, budget_s, counts):
    """The oracle (numpy restatement of the reference) on a bounded sample of
    the same matvec: the far field of one Morton-contiguous block of level-3
    subtrees holding 1/k of the modelled far-field work (the multi-GPU
    partition of k parts, part 0), and every k-th near-field target group /
    correction entry; the sample time is scaled by k."""
    import oracle
    from paper_2408_02274_b200.partition import level3_partition
    tree, hier, smap, mom, cp = inputs
    op = oracle.OperatorData(disc, mats, smap, mom, cp.ell_idx, cp.src_idx, tree, hier)
    # the numpy port runs ~1.5 GFLOP/s of the algorithmic count on 16 cores
    k = max(1, int(round(counts["total"] / 1.5e9 / budget_s)))
    k = min(k, tree.level(3).n_boxes)
    part = level3_partition(tree, hier, k, disc.n_patches, disc.n_c)[0]
    ranges = {d: part.levels[d]["box"] for d in part.levels}
    t0 = time.perf_counter()
    oracle.muller_apply(op, y, stride=k, box_ranges=ranges)
    wall = time.perf_counter() - t0
    est = wall * k
    cores = os.cpu_count()
    return {"value": 4 * disc.n_points / est, "unit": "unknowns*matvec/s",
            "cores": cores, "kind": "port",
            "sample": (f"oracle/ (numpy restatement of the reference): far field of "
                       f"level-3 subtrees {part.box3} (1/{k} of the modelled work), "
                       f"every {k}-th near-field box / patch group / correction entry; "
                       f"sample wall {wall:.1f}s x{k} = estimated full matvec {est:.1f}s; "
                       f"numpy/OpenBLAS threads={os.environ.get('OPENBLAS_NUM_THREADS', cores)}")}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np  # noqa: F401
    disc, mats, y, name = workload(args.n_refine, args.k0_pi, args.geometry)
    inputs = plan_inputs(disc, mats)
    counts = work_counts(inputs[0], inputs[1])
    per_step = min(15.0, 150.0 / max(1, args.steps + args.warmup))
    vals = []
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(disc, mats, y, inputs, per_step, counts)
        if i >= args.warmup:
            vals.append(cb)
    v = statistics.mean(c["value"] for c in vals)
    t_step = 4 * disc.n_points / v
    line = {"impl": "reference", "metric": "IFGF N-Muller matvec unknowns*matvec/s",
            "value": v, "unit": "unknowns*matvec/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c128/f64", "data": "synthetic (seeded N(0,1) densities)",
            "config": {"workload": name, "unknowns": 4 * disc.n_points,
                       "parallelism": "cpu"},
            "cpu_baseline": {**vals[-1], "value": v},
            "e2e": {"value": v, "unit": "unknowns*matvec/s",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2408_02274_b200.build import build
    from paper_2408_02274_b200.engine import kernel_times, set_kernel_timing
    from paper_2408_02274_b200.operator import MullerOperator

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    use_part = world > 1 or args.force_partition
    if use_part:
        # keep rank 0's stdout to the one JSON line (NCCL prints its version
        # banner at NCCL_DEBUG=VERSION/INFO; an explicit setting is kept)
        os.environ.setdefault("NCCL_DEBUG", "WARN")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        build()
    if world > 1:
        dist.barrier()
    disc, mats, y, name = workload(args.n_refine, args.k0_pi, args.geometry)
    t0 = time.time()
    inputs = plan_inputs(disc, mats, args.device_moments)
    tree, hier, smap, mom, cp = inputs
    op = MullerOperator(disc, mats, smap, mom, (cp.ell_idx, cp.src_idx),
                        tree=tree, hierarchy=hier)
    counts = work_counts(tree, hier)
    runner = op
    if use_part:
        # partitioned matvec: Morton level-3 subtrees per rank, NCCL sums
        from paper_2408_02274_b200.octree import accumulation_plan
        from paper_2408_02274_b200.partition import (DistributedMullerOperator,
                                                     level3_partition)
        parts = level3_partition(tree, hier, world, disc.n_patches, disc.n_c)
        runner = DistributedMullerOperator(op, parts[rank])
        mine = 0
        for d in range(4, tree.depth + 1):
            ap = accumulation_plan(tree, hier, d, geometry=False)
            lo, hi = parts[rank].levels[d - 1]["seg"]
            mine += W_PROP * int(ap.inst_off[hi] - ap.inst_off[lo]) + W_COEF * (hi - lo)
        counts = dict(counts, prop=mine)
    t_plan = time.time() - t0
    dev = torch.device("cuda", local)
    yd = torch.from_numpy(y).to(dev)
    out = torch.empty_like(yd)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(max(args.warmup, 3)):
        runner.apply_device(yd, out)
    torch.cuda.synchronize()
    launches_per_step = runner.last_launches()
    # ---- timed device loop (events per step, L2 flushed between steps)
    set_kernel_timing(op.plan, True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record()
            runner.apply_device(yd, out)
            evs[i][1].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_steps = [a.elapsed_time(b) for a, b in evs]
    ms = sum(ms_steps) / len(ms_steps)
    ktimes = kernel_times(op.plan)
    set_kernel_timing(op.plan, False)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # ---- end to end through the host API
    y_host = np.ascontiguousarray(y)
    if not use_part:
        host_apply = op.apply                 # library host path (pinned staging)
    else:
        y_pin = torch.from_numpy(y_host).pin_memory()
        o_pin = torch.empty_like(y_pin).pin_memory()

        def host_apply(v):
            y_pin.copy_(torch.from_numpy(v))
            yd.copy_(y_pin, non_blocking=True)
            runner.apply_device(yd, out)
            o_pin.copy_(out, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            return o_pin.numpy().copy()
    host_apply(y_host)
    e2e_t = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        host_apply(y_host)
        e2e_t.append(time.perf_counter() - t)
    e2e_s = sum(e2e_t) / len(e2e_t)
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    clocks = clk.summary()
    if rank != 0:
        if use_part:
            dist.barrier()
            dist.destroy_process_group()
        return
    unknowns = 4 * disc.n_points
    value = unknowns / (ms * 1e-3)        # one matvec over all ranks
    prop_ms, prop_n = ktimes["propagate"]
    prop_flop = counts["prop"] * args.steps
    achieved = prop_flop / (prop_ms * 1e-3) / 1e12 if prop_ms > 0 else None
    traffic = None
    tf = ROOT / "profiles" / f"traffic_n{args.n_refine}.json"
    if args.geometry != "sphere":
        tf = ROOT / "profiles" / f"traffic_{args.geometry}_n{args.n_refine}.json"
    if tf.exists() and args.k0_pi is None:
        traffic = json.loads(tf.read_text()).get("propagate_bytes_per_launch")
    kern = {k: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps}
            for k, v in ktimes.items() if v[1]}
    line = {
        "metric": "IFGF N-Muller matvec unknowns*matvec/s", "value": value,
        "unit": "unknowns*matvec/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128/f64",
        "data": "synthetic (seeded N(0,1) densities; analytic sphere mesh)",
        "config": {"workload": name, "unknowns": unknowns, "points": disc.n_points,
                   "depth": tree.depth, "segments": int(sum(hier.level(d).n_segments
                                                            for d in hier.cone_levels)),
                   "algorithmic_gflop_per_matvec": counts["total"] / 1e9,
                   "l2": "flushed (256 MB write) before every timed step",
                   "parallelism": (f"morton-level3-partition x{world} (NCCL all-reduce "
                                   "of far field + result)") if use_part else "single-gpu",
                   "plan_build_s": round(t_plan, 1),
                   "geometry_on_device_levels": sorted(getattr(op.plan, "otf_levels", [])),
                   "stream_parts": int(getattr(op.plan, "stream_parts", 1) or 1)},
        "roofline": {"kernel": "propagate (K4: child->parent re-interpolation on "
                               "FP64 DMMA + fused K3)",
                     "bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                     "unit": "TFLOP/s", "frac": (achieved / FP64_PEAK_TFLOPS
                                                 if achieved else None),
                     "traffic": traffic,
                     "flop_per_launch": counts["prop"] / max(1, prop_n // args.steps),
                     "ms_per_launch": prop_ms / max(1, prop_n),
                     "peak_source": "FP64 mma.sync m8n8k4 measured on B200 "
                                    "(tools/fp64_peak.cu, profiles/fp64_peak_r01.txt); "
                                    "MEASURED_PEAKS.json has no FP64 entry",
                     "share_of_step": prop_ms / args.steps / ms},
        "kernels": kern,
        "e2e": {"value": unknowns / e2e_s, "unit": "unknowns*matvec/s",
                "h2d_bytes_per_step": unknowns * 16, "d2h_bytes_per_step": unknowns * 16},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline and not args.device_moments:
        line["cpu_baseline"] = cpu_baseline(disc, mats, y, inputs, 15.0, counts)
    if world == 1 and not args.no_gmres:
        line["gmres"] = gmres_cfg1()
    print(json.dumps(line), flush=True)
    if use_part:
        dist.barrier()
        dist.destroy_process_group()


def gmres_cfg1():
    """BASELINE cfg 1 GMRES: sphere (2,10), k0 = 2 pi, tol 1e-6, x-polarised
    plane wave exp(i k0 z); reference: 38 iterations, 719-762 s on 8 cores."""
    import numpy as np
    from paper_2408_02274_b200 import surface
    from paper_2408_02274_b200.fields import plane_wave
    from paper_2408_02274_b200.operator import MaterialPair, build_muller_operator
    from paper_2408_02274_b200.solver import gmres
    disc = surface.make_sphere_surface(2, 10)
    k0 = 2 * np.pi
    op = build_muller_operator(disc, MaterialPair(1.0, 1.0, 2.25, 1.0, k0))
    b = op.rhs(plane_wave(k0, direction=(0.0, 0.0, 1.0), polarization=(1.0, 0.0, 0.0),
                          omega=k0))
    gmres(op, b, tol=1e-6, max_iter=300)
    x, rep = gmres(op, b, tol=1e-6, max_iter=300)
    return {"config": "cfg1 sphere(2,10) k0=2pi eps_r=2.25, tol 1e-6", "iterations":
            rep.iterations, "final_residual": rep.residuals[-1], "solve_s": rep.wall_time}


def rss_watchdog(limit_gb: float):
    """Kill this process (only) before the host runs out of memory."""
    import threading

    def watch():
        while True:
            try:
                with open(f"/proc/{os.getpid()}/status") as fh:
                    for line in fh:
                        if line.startswith("VmRSS:"):
                            kb = int(line.split()[1])
                            if kb > limit_gb * 1024 * 1024:
                                sys.stderr.write(f"RSS {kb / 1e6:.1f} GB > limit, abort\n")
                                sys.stderr.flush()
                                os.kill(os.getpid(), 9)
            except Exception:
                pass
            time.sleep(0.5)

    threading.Thread(target=watch, daemon=True).start()


def main():
    args = parse()
    if args.max_rss_gb > 0:
        rss_watchdog(args.max_rss_gb)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
