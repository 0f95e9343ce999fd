"""Reference-side GMRES residual history on a PATCHGRID geometry (build
container only: imports the unmodified reference from /root/reference).
Used to tell reference properties from port defects (DESIGN 9).

  python tools/ref_gmres_patchgrid.py tests/golden/sl1.patchgrid 10 2.0 12.11 15
"""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import emscat.geometry as rg  # noqa: E402
from emscat.operators import MaterialPair, build_muller_operator  # noqa: E402
from emscat.reference import plane_wave  # noqa: E402
from emscat.solver import gmres  # noqa: E402

path, nc, k0pi, eps, iters = sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
disc = rg.load_surface(path, nc)
k0 = k0pi * np.pi
mats = MaterialPair(1.0, 1.0, eps, 1.0, k0)
t0 = time.time()
op = build_muller_operator(disc, mats)
print("plan", time.time() - t0, flush=True)
b = op.rhs(plane_wave(k0, direction=(0.0, 1.0, 0.0), polarization=(0.0, 0.0, 1.0), omega=k0))
t0 = time.time()
x, rep = gmres(op.apply, b, tol=1e-12, max_iter=iters)
print("residuals", [round(float(r), 4) for r in rep.residuals], "time", time.time() - t0, flush=True)
