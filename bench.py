#!/usr/bin/env python
"""Benchmark: IFGF-accelerated N-Muller matvec throughput on B200.

metric  = unknowns * matvec / s  (4N unknowns per apply, BASELINE.json)
value   = device throughput with y resident in HBM (CUDA events, L2 flushed
          between steps)
e2e     = same metric through the public host API (MullerOperator.apply on a
          numpy vector: pinned staging, H2D, apply, D2H inside the timed call)

Default workload: BASELINE.json configs[4] (cfg 5, the north-star config):
unit dielectric sphere, eps_r = 2.25, k0 = 32 pi, 6 x 45^2 patches on 10x10
Chebyshev grids = 1,215,000 points = 4,860,000 unknowns; y ~ N(0,1) +
i N(0,1) (seed 0); the reference's default IFGF parameters.  Other configs:
--n-refine / --k0-pi (cfg 1 / 2 family), --geometry superellipsoid|slab
(cfg 3 / 4).

--impl reference: the reference algorithm's CPU implementation (the numpy
oracle restatement, `oracle/`: the reference is Python and cannot be
compiled) on this host's cores.  The cfg-5 plan alone takes ~10 min of host
numpy and a matvec hours, so the arm times one FULL matvec of the runnable
sphere(4,10) (k0 = 4 pi) and bounded samples of it per step, and reports the
workload's value as its algorithmic work / the port's achieved GFLOP/s
(labelled "extrapolated").

Multi-GPU (torchrun, N > 1): one process per GPU; rank r builds and runs
only its window of level-3 subtrees (far-field sources) and its target rows
(near field), exchanging one NCCL reduce-scatter of the far-field partials
and one all-gather of the result rows per matvec (partition.py).  The timed
region is barrier-bracketed and the max over ranks is reported.
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

FP64_PEAK_TFLOPS = 37.0   # DMMA m8n8k4 f64, measured (profiles/fp64_peak_r02.txt)
W_PROP = 75 * 75 * 16 * 4          # FLOP per (parent segment, child) instance
SEG_BYTES = 19_456                 # one segment's coefficients in HBM (80 x 16 complex, padded)
W_COEF = 16 * (3 * 3 * 25 + 5 * 5 * 15 + 5 * 5 * 15) * 4   # K3 per segment
W_EMIT = 2 * 75 * 16 * 4           # per (box, target) pair, x and x + h n
W_LEAF = 128                       # per (node, source) pair (2 kernels x 8 ch)
METRIC = "IFGF N-Muller matvec unknowns*matvec/s"
COUNTS_FILE = ROOT / "profiles" / "work_counts.json"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--n-refine", type=int, default=45)
    ap.add_argument("--k0-pi", type=float, default=None,
                    help="k0 / pi (sphere default: 32 at n_refine 45 (cfg 5), else n_refine)")
    ap.add_argument("--geometry", choices=["sphere", "superellipsoid", "slab"],
                    default="sphere", help="BASELINE cfg 1/2/5, cfg 3, cfg 4 bodies")
    ap.add_argument("--moments", choices=["auto", "host", "device"], default="auto",
                    help="singular moments: host restatement (reference-exact) or the "
                         "plan-time GPU kernel; auto = device above 100k points")
    ap.add_argument("--device-moments", action="store_true", help="= --moments device")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gmres", action="store_true")
    ap.add_argument("--max-rss-gb", type=float, default=0.0,
                    help="abort (kill this process) if host RSS exceeds this")
    ap.add_argument("--force-partition", action="store_true",
                    help="run the multi-GPU (rank) operator and NCCL exchange even at N=1")
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="one GPU: build and time only rank --emulate-rank's share of an "
                         "R-way partition (per-rank work / memory; no exchange)")
    ap.add_argument("--emulate-rank", type=int, default=0)
    args = ap.parse_args()
    if args.device_moments:
        args.moments = "device"
    if args.k0_pi is None and args.geometry == "sphere":
        args.k0_pi = 32.0 if args.n_refine == 45 else float(args.n_refine)
    return args


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload(n_refine, k0_pi=None, geometry="sphere"):
    """BASELINE configs: 'sphere' = cfg 1/2/5 family (sphere(n, 10), eps_r
    2.25; cfg 5 is n = 45 at k0 = 32 pi); 'superellipsoid' = cfg 3 (|x/2|^4 +
    |y|^4 + |z/0.5|^4 = 1, n x n subpatches per face on 12 x 12 grids, eps_r
    4, 2a = 8 wavelengths -> k0 = 4 pi); 'slab' = cfg 4 (exponent-8
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
        if n_refine == 45 and k0_pi == 32:
            name = "cfg5 " + name
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


def use_device_moments(args, disc) -> bool:
    return args.moments == "device" or (args.moments == "auto" and disc.n_points > 100_000)


def _stage_logger():
    t0 = time.time()
    return lambda what: print(f"[plan] {what} {time.time() - t0:.1f}s", file=sys.stderr,
                              flush=True)


def plan_inputs(disc, mats, device_moments=False, device_plan=False):
    """Host plan; device_plan: cone hierarchy and propagation types from the
    native device builder (csrc/planbuild.cu; integers identical to the host
    builder, tests/test_gpu_planbuild.py)."""
    from paper_2408_02274_b200 import nearfield, octree
    kmax = max(abs(mats.kappa_e), abs(mats.kappa_i))
    stage = _stage_logger()
    tree = octree.build_box_tree(disc.points, kmax)
    stage("tree")
    hier = octree.build_cone_hierarchy(tree, device=device_plan)
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
    stage("corrections")
    return tree, hier, smap, mom, cp


def work_counts(tree, hier):
    """Algorithmic FLOP per matvec from the plan (or a
    window's plan: that rank's share)."""
    from paper_2408_02274_b200 import octree
    D = tree.depth
    prop, pbytes, ninst = {}, {}, {}
    for d in range(4, D + 1):
        ap = octree.accumulation_plan(tree, hier, d, geometry=False)
        ninst[d] = int(ap.n_instances)
        prop[d] = W_PROP * ap.n_instances + W_COEF * hier.level(d - 1).n_segments
        # algorithmic HBM bytes of K4: child level read once, parent written once
        pbytes[d] = SEG_BYTES * (hier.level(d).n_segments + hier.level(d - 1).n_segments)
    cl, lvl = hier.level(D), tree.level(D)
    leaf = W_LEAF * 75 * int((cl.seg_off[1:] - cl.seg_off[:-1]) @ lvl.pt_count)
    emit = W_EMIT * sum(hier.level(d).cpt_idx.size for d in range(3, D + 1))
    return {"prop_by_level": prop, "prop": sum(prop.values()), "leaf": leaf,
            "instances_by_level": ninst,
            "prop_bytes": sum(pbytes.values()),
            "leaf_coef": W_COEF * cl.n_segments, "emit": emit,
            "total": sum(prop.values()) + leaf + W_COEF * cl.n_segments + emit}


def record_counts(name, counts, unknowns):
    """Keep the workload's algorithmic work where the reference arm (which
    cannot build the cfg-5 plan in minutes) finds it."""
    try:
        data = json.loads(COUNTS_FILE.read_text()) if COUNTS_FILE.exists() else {}
        entry = {"total_flop": counts["total"], "prop_flop": counts["prop"],
                 "unknowns": unknowns}
        if data.get(name) != entry:
            data[name] = entry
            COUNTS_FILE.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
    except OSError:
        pass


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


def _threads():
    return os.environ.get("OPENBLAS_NUM_THREADS", str(os.cpu_count()))


def oracle_sample(disc, mats, y, inputs, counts, budget_s, rate_guess=1.5e9):
    """Time the oracle (numpy restatement of the reference) on a bounded
    sample of one matvec: the far field of every `stride`-th box of level-3
    subtree block 0 (1/k of the subtrees), every k*stride-th near-field
    box / moment / correction entry.  Returns (sample wall s, sampled
    fraction of the matvec, description)."""
    import oracle
    from paper_2408_02274_b200.partition import level3_partition
    tree, hier, smap, mom, cp = inputs
    op = oracle.OperatorData(disc, mats, smap, mom, cp.ell_idx, cp.src_idx, tree, hier)
    frac = min(1.0, budget_s * rate_guess / counts["total"])
    n3 = tree.level(3).n_boxes
    k = max(1, min(n3, int(round(1.0 / frac))))
    stride = max(1, int(round(1.0 / (frac * k))))
    parts = level3_partition(tree, hier, k, disc.n_patches, disc.n_c)
    part = parts[0]
    ranges = {d: part.levels[d]["box"] for d in part.levels}
    t0 = time.perf_counter()
    oracle.muller_apply(op, y, stride=k * stride, box_ranges=ranges, far_stride=stride)
    wall = time.perf_counter() - t0
    sampled = part.work / max(1e-300, sum(p.work for p in parts)) / stride
    desc = (f"oracle/ (numpy restatement of the reference): far field of every "
            f"{stride}-th box of level-3 subtrees {part.box3} ({sampled:.2e} of the "
            f"modelled far-field work), every {k * stride}-th near-field box / moment / "
            f"correction entry; sample wall {wall:.1f}s")
    return wall, sampled, desc


def _oracle_full(disc, mats, y, inputs):
    import oracle
    tree, hier, smap, mom, cp = inputs
    op = oracle.OperatorData(disc, mats, smap, mom, cp.ell_idx, cp.src_idx, tree, hier)
    t0 = time.perf_counter()
    oracle.muller_apply(op, y)
    return time.perf_counter() - t0


def cpu_baseline(disc, mats, y, inputs, budget_s, counts):
    """The oracle (numpy restatement of the reference) on the host cores.
    Workloads whose full matvec fits the budget are timed whole.  Larger ones
    (cfg 5: ~97 TFLOP, hours of numpy) are timed as ONE full oracle matvec of
    cfg 1 (74 GFLOP, ~15 s) and scaled by algorithmic work: the port's time
    tracks its algorithmic FLOP.  A strided box sample
    of cfg 5 itself was tried and overstates the time ~6x (per-box Python
    overheads of tiny sampled boxes; profiles/bench_r02_cfg5_l1kernel.json)."""
    if counts["total"] <= 4e9 * budget_s:
        wall = _oracle_full(disc, mats, y, inputs)
        return {"value": 4 * disc.n_points / wall, "unit": "unknowns*matvec/s",
                "cores": os.cpu_count(), "kind": "port",
                "sample": f"one full oracle/ matvec of this workload ({wall:.1f}s); "
                          f"numpy/OpenBLAS threads={_threads()}"}
    cdisc, cmats, cy, cname = workload(2, 2.0, "sphere")
    cin = plan_inputs(cdisc, cmats)
    ccounts = work_counts(cin[0], cin[1])
    wall = _oracle_full(cdisc, cmats, cy, cin)
    rate = ccounts["total"] / wall
    est = counts["total"] / rate
    return {"value": 4 * disc.n_points / est, "unit": "unknowns*matvec/s",
            "cores": os.cpu_count(), "kind": "port", "extrapolated": True,
            "sample": f"one full oracle/ (numpy restatement of the reference) matvec of "
                      f"cfg 1 {cname} ({ccounts['total'] / 1e9:.1f} GFLOP in {wall:.1f}s = "
                      f"{rate / 1e9:.2f} GFLOP/s); this workload's "
                      f"{counts['total'] / 1e9:.0f} GFLOP at that rate = {est:.0f}s per "
                      f"matvec; numpy/OpenBLAS threads={_threads()}"}


def run_reference(args):
    """The reference arm (see module docstring): one full port matvec of
    sphere(4,10) as calibration, then warmup + steps bounded samples of it;
    value = the workload's algorithmic work at the port's achieved rate."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    _, _, _, name = workload(args.n_refine, args.k0_pi, args.geometry)
    counts_all = json.loads(COUNTS_FILE.read_text()) if COUNTS_FILE.exists() else {}
    target = counts_all.get(name)
    cal_disc, cal_mats, cal_y, cal_name = workload(4, 4.0, "sphere")
    stage = _stage_logger()
    inputs = plan_inputs(cal_disc, cal_mats)
    cal_counts = work_counts(inputs[0], inputs[1])
    stage("calibration plan")
    if target is None:            # a workload the arm can plan itself
        disc, mats, y, name = workload(args.n_refine, args.k0_pi, args.geometry)
        if disc.n_points > 100_000:
            print(json.dumps({"impl": "reference", "unavailable":
                              f"no recorded work count for {name} (run the b200 arm once)"}))
            return
        tin = plan_inputs(disc, mats)
        target = {"total_flop": work_counts(tin[0], tin[1])["total"],
                  "unknowns": 4 * disc.n_points}
    import oracle
    op = oracle.OperatorData(cal_disc, cal_mats, inputs[2], inputs[3], inputs[4].ell_idx,
                             inputs[4].src_idx, inputs[0], inputs[1])
    t0 = time.perf_counter()
    oracle.muller_apply(op, cal_y)
    t_full = time.perf_counter() - t0
    rate_full = cal_counts["total"] / t_full
    stage(f"full port matvec {t_full:.1f}s")
    per_step = min(10.0, 120.0 / max(1, args.steps + args.warmup))
    rates, walls, desc = [], [], ""
    for i in range(args.warmup + args.steps):
        wall, frac, desc = oracle_sample(cal_disc, cal_mats, cal_y, inputs, cal_counts,
                                         per_step, rate_full)
        if i >= args.warmup:
            rates.append(frac * cal_counts["total"] / wall)
            walls.append(wall)
    rate = rate_full               # the full measured matvec's rate
    t_target = target["total_flop"] / rate
    v = target["unknowns"] / t_target
    line = {"impl": "reference", "metric": METRIC, "value": v,
            "unit": "unknowns*matvec/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": statistics.mean(walls) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "c128/f64", "data": "synthetic (seeded N(0,1) densities)",
            "extrapolated": True,
            "config": {"workload": name, "unknowns": target["unknowns"],
                       "parallelism": "cpu",
                       "algorithmic_gflop_per_matvec": target["total_flop"] / 1e9,
                       "step": f"one bounded sample of a {cal_name} port matvec "
                               f"(ms_per_step = its wall time)"},
            "calibration": {"workload": cal_name, "full_matvec_s": t_full,
                            "gflop": cal_counts["total"] / 1e9,
                            "achieved_gflops": rate_full / 1e9,
                            "sampled_gflops": statistics.mean(rates) / 1e9},
            "cpu_baseline": {"value": v, "unit": "unknowns*matvec/s",
                             "cores": os.cpu_count(), "kind": "port",
                             "sample": f"one full {cal_name} port matvec ({t_full:.1f}s = "
                                       f"{rate_full / 1e9:.2f} GFLOP/s of its algorithmic "
                                       f"work); value = {target['total_flop'] / 1e9:.0f} "
                                       f"GFLOP at that rate; steps: {desc}; numpy/OpenBLAS "
                                       f"threads={_threads()}"},
            "e2e": {"value": v, "unit": "unknowns*matvec/s",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _traffic(name):
    """Per-launch DRAM bytes of K4 from an ncu --set full capture of this
    workload (profiles/traffic_*.json), if one was committed."""
    for f in sorted((ROOT / "profiles").glob("traffic_*.json")):
        try:
            d = json.loads(f.read_text())
        except (OSError, ValueError):
            continue
        if d.get("workload") == name:
            return d.get("propagate_bytes_per_launch"), f.name
    return None, None


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2408_02274_b200.build import build
    from paper_2408_02274_b200 import engine
    from paper_2408_02274_b200.engine import kernel_times, level_times, set_kernel_timing
    from paper_2408_02274_b200.operator import MullerOperator

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    use_rank = world > 1 or args.force_partition
    emulate = args.emulate_ranks > 0
    if use_rank:
        # keep rank 0's stdout to the one JSON line (NCCL prints its version
        # banner at NCCL_DEBUG=VERSION/INFO; an explicit setting is kept)
        os.environ.setdefault("NCCL_DEBUG", "WARN")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        build()
    if world > 1:
        dist.barrier()
    disc, mats, y, name = workload(args.n_refine, args.k0_pi, args.geometry)
    dev_mom = use_device_moments(args, disc)
    t0 = time.time()
    inputs = None
    if use_rank or emulate:
        from paper_2408_02274_b200 import octree
        from paper_2408_02274_b200.partition import (DistributedMullerOperator,
                                                     level3_partition)
        kmax = max(abs(mats.kappa_e), abs(mats.kappa_i))
        tree = octree.build_box_tree(disc.points, kmax)
        n_r, r = (args.emulate_ranks, args.emulate_rank) if emulate else (world, rank)
        part = level3_partition(tree, None, n_r, disc.n_patches, disc.n_c)[r]
        runner = DistributedMullerOperator(disc, mats, part, tree=tree,
                                           exchange=False if emulate else None,
                                           device_moments=dev_mom, device_plan=dev_mom)
        op = runner.op
        counts = work_counts(runner.view, runner.hier)
    else:
        inputs = plan_inputs(disc, mats, dev_mom, device_plan=dev_mom)
        tree, hier, smap, mom, cp = inputs
        op = MullerOperator(disc, mats, smap, mom, (cp.ell_idx, cp.src_idx),
                            tree=tree, hierarchy=hier)
        runner = op
        counts = work_counts(tree, hier)
        record_counts(name, counts, 4 * disc.n_points)
    t_plan = time.time() - t0
    dev = torch.device("cuda", local)
    yd = torch.from_numpy(y).to(dev)
    out = torch.empty_like(yd)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        if emulate:       # this rank's far + near work; no exchange
            runner.far_phase(yd)
            c = runner.xfar_mine.numel()
            runner.xfar_mine.copy_(runner.xfar[r * c:(r + 1) * c])
            runner.near_phase(yd)
        else:
            runner.apply_device(yd, out)

    for _ in range(max(args.warmup, 3)):
        step()
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
            step()
            evs[i][1].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_steps = [a.elapsed_time(b) for a, b in evs]
    ms = sum(ms_steps) / len(ms_steps)
    ktimes = kernel_times(op.plan)
    ltimes = level_times(op.plan)
    set_kernel_timing(op.plan, False)
    rank_info = {"ms": ms, "plan_s": t_plan, "device_gib": op.plan.device_bytes() / 2**30,
                 "prop_gflop": counts["prop"] / 1e9, "total_gflop": counts["total"] / 1e9}
    if world > 1:
        t = torch.tensor([ms, t_plan], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, t_plan = float(t[0].item()), float(t[1].item())
        gathered = [None] * world
        dist.all_gather_object(gathered, rank_info)
        rank_info = gathered
        tot = torch.tensor([counts["total"]], dtype=torch.float64, device=dev)
        dist.all_reduce(tot)
        total_flop = float(tot.item())
    else:
        total_flop = counts["total"]
    # ---- end to end through the host API
    y_host = np.ascontiguousarray(y)
    if not (use_rank or emulate):
        host_apply = op.apply                 # library host path (pinned staging)
    else:
        y_pin = torch.from_numpy(y_host).pin_memory()
        o_pin = torch.empty_like(y_pin).pin_memory()

        def host_apply(v):
            y_pin.copy_(torch.from_numpy(v))
            yd.copy_(y_pin, non_blocking=True)
            step()
            o_pin.copy_(out, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            return o_pin.numpy().copy()
    host_apply(y_host)
    e2e_t = []
    for _ in range(args.steps if not emulate else 0):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        host_apply(y_host)
        e2e_t.append(time.perf_counter() - t)
    e2e_s = sum(e2e_t) / len(e2e_t) if e2e_t else ms * 1e-3
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    clocks = clk.summary()
    if rank != 0:
        if use_rank:
            dist.barrier()
            dist.destroy_process_group()
        return
    unknowns = 4 * disc.n_points
    value = unknowns / (ms * 1e-3)        # one matvec over all ranks
    prop_ms, prop_n = ktimes["propagate"]
    achieved = counts["prop"] * args.steps / (prop_ms * 1e-3) / 1e12 if prop_ms > 0 else None
    traffic, tsrc = _traffic(name)
    kern = {k: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps}
            for k, v in ktimes.items() if v[1]}
    par = "single-gpu"
    if use_rank:
        par = (f"{world} ranks: level-3 subtree windows (sources) + target rows, "
               "NCCL reduce-scatter of far partials + all-gather of result rows")
    if emulate:
        par = (f"emulated rank {args.emulate_rank} of {args.emulate_ranks} on one GPU "
               "(its share of the work only; no exchange)")
    line = {
        "metric": METRIC, "value": value,
        "unit": "unknowns*matvec/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128/f64",
        "data": "synthetic (seeded N(0,1) densities; analytic sphere mesh)",
        "config": {"workload": name, "unknowns": unknowns, "points": disc.n_points,
                   "depth": tree.depth,
                   "algorithmic_gflop_per_matvec": total_flop / 1e9,
                   "l2": "flushed (256 MB write) before every timed step",
                   "parallelism": par,
                   "moments": ("device kernel, exact mode (host graded nodes, reference "
                               "operation order: beta_s/beta_d to rounding, apply parity "
                               "< 1e-10 at c1/c2n4, tests/test_gpu_moments.py)" if dev_mom else
                               "host restatement (reference-exact)"),
                   "plan_builder": ("device (cones + propagation types, "
                                    "csrc/planbuild.cu)" if dev_mom else "host numpy"),
                   "plan_build_s": round(t_plan, 1),
                   "device_plan_gib": round(op.plan.device_bytes() / 2**30, 2),
                   "geometry_on_device_levels": sorted(getattr(op.plan, "otf_levels", [])),
                   "geometry_on_device_mode": (
                       "in the propagation kernel (IFGFB_OTF_PRE_MB=0)"
                       if os.environ.get("IFGFB_OTF_PRE_MB", "").strip() == "0"
                       else "node tables per chunk of parent rows (otf_tables_kernel) "
                            "ahead of each propagation launch; timed inside propagate"),
                   "k4_tiles": ("formed on the device (no tile records)"
                                if getattr(op.plan, "tile_free", False) else "host records"),
                   "k4_kernel": engine.k4_mode(),
                   "stream_parts": int(getattr(op.plan, "stream_parts", 1) or 1)},
        "roofline": {"kernel": "propagate (K4: child->parent re-interpolation on "
                               "FP64 DMMA + fused K3)" + (" of rank 0" if world > 1 else ""),
                     "bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                     "unit": "TFLOP/s", "frac": (achieved / FP64_PEAK_TFLOPS
                                                 if achieved else None),
                     "traffic": traffic, "traffic_source": tsrc,
                     "traffic_algorithmic": counts["prop_bytes"] / max(1, prop_n // args.steps),
                     "flop_per_launch": counts["prop"] / max(1, prop_n // args.steps),
                     "ms_per_launch": prop_ms / max(1, prop_n),
                     "peak_source": "FP64 mma.sync m8n8k4 measured on B200 at 1965 MHz "
                                    "(tools/fp64_peak.cu, profiles/fp64_peak_r02.txt with "
                                    "its clock record); MEASURED_PEAKS.json has no FP64 entry",
                     "share_of_step": prop_ms / args.steps / ms,
                     "by_level": {
                         str(d): {"ms_per_step": round(t / args.steps, 3),
                                  "tflops": (round(counts["prop_by_level"][d] * args.steps
                                                   / (t * 1e-3) / 1e12, 2)
                                             if t > 0 and d in counts["prop_by_level"] else None),
                                  "geometry_on_device": d in getattr(op.plan, "otf_levels", [])}
                         for d, (t, _n) in sorted(ltimes.items())}},
        "kernels": kern,
        "e2e": {"value": unknowns / e2e_s, "unit": "unknowns*matvec/s",
                "h2d_bytes_per_step": unknowns * 16 * world,
                "d2h_bytes_per_step": unknowns * 16 * world},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
    }
    otf = sorted(getattr(op.plan, "otf_levels", []))
    if otf and os.environ.get("IFGFB_OTF_PRE_MB", "").strip() != "0":
        # node tables of the on-device-geometry levels: written by the pre-pass
        # and read back by the propagation, 75 nodes x 56 B per instance
        extra = 2 * 75 * 56 * sum(counts["instances_by_level"].get(d, 0) for d in otf)
        line["roofline"]["traffic_prepass_tables"] = extra / max(1, prop_n // args.steps)
        line["roofline"]["traffic_note"] = (
            "traffic: ncu launch list captured before the node-table pre-pass "
            "(profiles/launches_r02_cfg5_wide.csv); traffic_prepass_tables = the "
            f"pre-pass's table bytes on levels {otf} per K4 launch, computed from the "
            "plan (written once, read once), to be added to it")
    if world > 1 or emulate:
        line["ranks"] = rank_info if isinstance(rank_info, list) else [rank_info]
    if world == 1 and not emulate and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(disc, mats, y, inputs, 15.0, counts)
    if world == 1 and not emulate and not args.no_gmres:
        line["gmres"] = gmres_cfg1()
    print(json.dumps(line), flush=True)
    if use_rank:
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
