"""D_far parity diagnostics: GPU far field vs the reference golden."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import _support as S
from paper_2408_02274_b200.engine import ifgf_apply
for name in sys.argv[1:] or ["s1", "c1"]:
    z, inp = S.golden(name), S.inputs(name)
    out, od = ifgf_apply(inp["tree"], inp["hier"], z["weights"], inp["kappas"],
                         displaced_normals=inp["disc"].normals, displaced_step=1e-6)
    d_g = (od - out) / 1e-6
    d_r = (z["far_disp"] - z["far"]) / 1e-6
    print(name, "far rel %.2e disp rel %.2e D_far rel %.2e" % (S.rel(out, z["far"]), S.rel(od, z["far_disp"]), S.rel(d_g, d_r)),
          "bitwise-equal far:", np.mean(out == z["far"]), "disp:", np.mean(od == z["far_disp"]))
