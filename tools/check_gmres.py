import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2408_02274_b200 import surface
from paper_2408_02274_b200.operator import MaterialPair, build_muller_operator
from paper_2408_02274_b200.fields import plane_wave
from paper_2408_02274_b200.solver import gmres
z = np.load("tests/golden/c1_gmres.npz")
disc = surface.make_sphere_surface(2, 10)
k0 = 2 * np.pi
op = build_muller_operator(disc, MaterialPair(1.0, 1.0, 2.25, 1.0, k0))
b = op.rhs(plane_wave(k0, direction=(0.0, 0.0, 1.0), polarization=(1.0, 0.0, 0.0), omega=k0))
print("rhs rel", np.linalg.norm(b - z["b"]) / np.linalg.norm(z["b"]))
x, rep = gmres(op, b, tol=1e-6, max_iter=300)
x, rep = gmres(op, b, tol=1e-6, max_iter=300)
r_ref = z["residuals"]; r = np.array(rep.residuals)
print("iters", rep.iterations, int(z["iterations"]), "wall", rep.wall_time, "ref wall", float(z["wall"]))
if r.size == r_ref.size:
    print("history max rel diff", np.max(np.abs(r - r_ref) / r_ref))
print("x rel", np.linalg.norm(x - z["x"]) / np.linalg.norm(z["x"]))
true_res = np.linalg.norm(b - op.apply(x)) / np.linalg.norm(b)
print("true residual", true_res)
