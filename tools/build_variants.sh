#!/bin/bash
# build library variants for tools/ab_variants.sh: tools/build_variants.sh name "-DFLAG=.." ...
mkdir -p variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  python - "$name" "$flags" <<'PY'
import subprocess, sys
from paper_2408_02274_b200 import build as b
name, flags = sys.argv[1], sys.argv[2].split()
cmd = [b._nvcc(), *b.NVCC_FLAGS, *flags, "-o", f"variants/{name}.so", *[str(b.CSRC / s) for s in b.SOURCES]]
subprocess.run(cmd, check=True, cwd=b.CSRC.parent.parent)
PY
done
