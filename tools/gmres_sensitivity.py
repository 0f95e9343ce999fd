"""How much does the cfg-1 GMRES residual history move when every matvec is
perturbed at the reference's own rounding floor (rel 3e-11, its vec/seq
difference)?  That sets the honest parity floor for the history."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2408_02274_b200 import surface
from paper_2408_02274_b200.operator import MaterialPair, build_muller_operator
from paper_2408_02274_b200.fields import plane_wave
from paper_2408_02274_b200.solver import gmres
z = np.load("tests/golden/c1_gmres.npz")
disc = surface.make_sphere_surface(2, 10)
k0 = 2 * np.pi
op = build_muller_operator(disc, MaterialPair(1.0, 1.0, 2.25, 1.0, k0))
b = z["b"]
_, rep0 = gmres(op, b, tol=1e-6, max_iter=300)
r0 = np.array(rep0.residuals)
ref = z["residuals"]
print("device vs reference: rel", np.max(np.abs(r0 - ref) / ref), "abs", np.max(np.abs(r0 - ref)))
rng = np.random.default_rng(0)
for eps in (1e-11, 3e-11, 1e-10):
    class Noisy:
        def apply_device(self, v, out=None):
            o = op.apply_device(v, out)
            n = torch.from_numpy(rng.normal(size=(o.numel(), 2)) @ [1, 1j]).to(o.device)
            o += eps * torch.linalg.vector_norm(o) / np.sqrt(o.numel()) * n
            return o
    _, rep = gmres(Noisy(), b, tol=1e-6, max_iter=300)
    r = np.array(rep.residuals)
    m = min(r.size, r0.size)
    print(f"matvec noise {eps:.0e}: its {rep.iterations} history rel {np.max(np.abs(r[:m]-r0[:m])/r0[:m]):.2e} abs {np.max(np.abs(r[:m]-r0[:m])):.2e}")
