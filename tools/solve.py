#!/usr/bin/env python
"""GMRES solve on one B200 for a BASELINE configuration (the reference's
`solve` / `validate-sphere` commands, reference cli.py:230-289, on the
device path): plan build, right-hand side from the configuration's incident
field, device GMRES (solver.gmres), and for the sphere the interior-field
error against the Mie series at 1,000 points (radius 0.7).

  python tools/solve.py --geometry sphere --n-refine 2            # cfg 1
  python tools/solve.py --geometry superellipsoid --n-refine 8 --tol 1e-5   # cfg 3
  python tools/solve.py --geometry slab --n-refine 3 --tol 1e-5   # cfg 4 (smaller)
  python tools/solve.py --n-refine 45 --k0-pi 32 --max-iter 50 --tol 1e-12 \
      --device-moments                                            # cfg 5, 50 iterations

Incident fields (BASELINE.json): sphere: x-polarised plane wave exp(i k0 z);
superellipsoid: plane wave from theta = 30 deg, phi = 45 deg, TE (E along
phi-hat); slab: complex-source Gaussian beam along +x (the long axis),
waist one wavelength, waist plane half a wavelength before the end.
Prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def incident_for(geometry, mats, disc):
    import numpy as np
    from paper_2408_02274_b200.fields import gaussian_beam, plane_wave
    k0 = float(np.real(mats.kappa_e))
    if geometry == "sphere":
        return plane_wave(k0, direction=(0.0, 0.0, 1.0), polarization=(1.0, 0.0, 0.0),
                          omega=mats.omega), "plane wave exp(i k0 z), x-pol"
    if geometry == "superellipsoid":
        th, ph = np.deg2rad(30.0), np.deg2rad(45.0)
        d = (np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th))
        pol = (-np.sin(ph), np.cos(ph), 0.0)
        return plane_wave(k0, direction=d, polarization=pol, omega=mats.omega), \
            "plane wave theta=30 phi=45 TE"
    lam = 2 * np.pi / k0
    x0 = disc.points[:, 0].min() - 0.5 * lam
    return gaussian_beam(k0, focus=(x0, 0.0, 0.0), direction=(1.0, 0.0, 0.0),
                         polarization=(0.0, 0.0, 1.0), waist=lam, omega=mats.omega), \
        "Gaussian beam along +x, z-pol, waist 1 wavelength at x_min - wavelength/2"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--geometry", choices=["sphere", "superellipsoid", "slab"], default="sphere")
    ap.add_argument("--n-refine", type=int, default=2)
    ap.add_argument("--k0-pi", type=float, default=None)
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--max-iter", type=int, default=500)
    ap.add_argument("--device-moments", action="store_true")
    ap.add_argument("--eps-r", type=float, default=None, help="override the config's eps_r")
    ap.add_argument("--incident", default="config", choices=["config", "plane-x", "plane-y", "plane-z"],
                    help="override the config's incident field with a plane wave along an axis")
    ap.add_argument("--stream-parts", type=int, default=None,
                    help="force single-GPU streaming over this many subtree groups")
    ap.add_argument("--geom-on-device", default=None, choices=["none", "all", "auto"],
                    help="propagation node geometry policy (engine._choose_otf)")
    args = ap.parse_args()

    import numpy as np
    import torch
    import bench
    from paper_2408_02274_b200.build import build
    from paper_2408_02274_b200.fields import evaluate_fields, fibonacci_sphere, mie_solution
    from paper_2408_02274_b200.operator import DensityBlock, MullerOperator
    from paper_2408_02274_b200.solver import gmres

    build()
    torch.cuda.set_device(0)
    disc, mats, _, name = bench.workload(args.n_refine, args.k0_pi, args.geometry)
    if args.eps_r is not None:
        from paper_2408_02274_b200.operator import MaterialPair
        mats = MaterialPair(1.0, 1.0, args.eps_r, 1.0, mats.omega)
        name += f" (eps_r overridden: {args.eps_r:g})"
    t0 = time.time()
    tree, hier, smap, mom, cp = bench.plan_inputs(disc, mats, args.device_moments)
    if args.geom_on_device:
        import os
        os.environ["IFGFB_GEOM_ON_DEVICE"] = args.geom_on_device
    op = MullerOperator(disc, mats, smap, mom, (cp.ell_idx, cp.src_idx), tree=tree,
                        hierarchy=hier, stream_parts=args.stream_parts)
    t_plan = time.time() - t0
    if args.incident == "config":
        inc, inc_name = incident_for(args.geometry, mats, disc)
    else:
        from paper_2408_02274_b200.fields import plane_wave
        ax = "xyz".index(args.incident[-1])
        dvec = np.eye(3)[ax]
        pol = np.eye(3)[(ax + 1) % 3]
        inc = plane_wave(float(np.real(mats.kappa_e)), direction=tuple(dvec),
                         polarization=tuple(pol), omega=mats.omega)
        inc_name = f"plane wave along {args.incident[-1]}"
    b = op.rhs(inc)
    # one matvec (warm) for the per-matvec time
    bd = torch.from_numpy(b).cuda()
    out = torch.empty_like(bd)
    op.apply_device(bd, out)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    op.apply_device(bd, out)
    ev1.record()
    torch.cuda.synchronize()
    t_mv = ev0.elapsed_time(ev1) / 1e3
    x, rep = gmres(op, b, tol=args.tol, max_iter=args.max_iter)
    line = {"workload": name, "unknowns": 4 * disc.n_points, "depth": tree.depth,
            "incident": inc_name, "tol": args.tol, "max_iter": args.max_iter,
            "plan_build_s": round(t_plan, 1), "matvec_s": t_mv,
            "otf_levels": sorted(getattr(op.plan, "otf_levels", [])),
            "residuals_head": [float(r) for r in rep.residuals[:12]],
            "gmres": {"iterations": rep.iterations, "converged": rep.converged,
                      "final_residual": float(rep.residuals[-1]) if rep.residuals else 0.0,
                      "solve_s": rep.wall_time,
                      "s_per_iteration": rep.wall_time / max(rep.iterations, 1)}}
    if args.geometry == "sphere":
        m, j = op.decode(x)
        dens = DensityBlock.from_currents(disc, j, m)
        pv = fibonacci_sphere(1000, 0.7)
        t1 = time.time()
        e, h = evaluate_fields(disc, dens, mats, pv, "interior")
        t_f = time.time() - t1
        e_ref, h_ref = mie_solution(1.0, mats)._eval(pv, "interior")
        line["validate_sphere"] = {
            "points": 1000, "radius": 0.7, "field_eval_s": t_f,
            "error_e": float(np.linalg.norm(e - e_ref) / np.linalg.norm(e_ref)),
            "error_h": float(np.linalg.norm(h - h_ref) / np.linalg.norm(h_ref))}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
