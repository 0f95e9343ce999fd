"""One small N-Muller apply (s1 golden, 2,400 unknowns) and one ifgf_apply,
for compute-sanitizer (racecheck / memcheck / synccheck) runs:

  compute-sanitizer --tool racecheck python tools/sanitize_apply.py

Both K4 variants run (IFGFB_K4 selects one per process; see far.cu)."""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    from _support import golden, inputs, rel
    from paper_2408_02274_b200.operator import MullerOperator
    z, inp = golden("s1"), inputs("s1")
    op = MullerOperator(inp["disc"], inp["mats"], inp["smap"], inp["moments"],
                        (inp["corr"].ell_idx, inp["corr"].src_idx), tree=inp["tree"],
                        hierarchy=inp["hier"], stream_parts=2)
    e_stream = rel(op.apply(z["y"]), z["apply_y"])
    op = MullerOperator(inp["disc"], inp["mats"], inp["smap"], inp["moments"],
                        (inp["corr"].ell_idx, inp["corr"].src_idx), tree=inp["tree"],
                        hierarchy=inp["hier"], geometry_on_device="all")
    e_otf = rel(op.apply(z["y"]), z["apply_y"])
    print(f"sanitize_apply: s1 apply vs reference {e_stream:.2e} (streamed), "
          f"{e_otf:.2e} (on-device geometry)")
    assert e_stream < 1e-10 and e_otf < 1e-10
    _ = np


if __name__ == "__main__":
    main()
