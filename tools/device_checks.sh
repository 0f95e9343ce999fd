#!/bin/bash
# Memory-safety run without compute-sanitizer (closed on this GPU pool):
# builds the library with -DIFGFB_DEVICE_CHECKS (bounds asserts in the K4
# staging, near-field lists; csrc/common.cuh IFGFB_DCHECK) and runs the GPU
# parity tests against it for every propagation kernel.  A violated check
# prints its condition and traps (the test then fails).
#   bash tools/device_checks.sh > profiles/device_checks_r02.log 2>&1
set -u
mkdir -p variants
python - <<'PY'
import subprocess
from paper_2408_02274_b200 import build as b
cmd = [b._nvcc(), *b.NVCC_FLAGS, "-DIFGFB_DEVICE_CHECKS", "-o", "variants/checked.so",
       *[str(b.CSRC / s) for s in b.SOURCES]]
subprocess.run(cmd, check=True, cwd=b.CSRC.parent.parent)
PY
for k4 in wide l1free l1 ringfree ring; do
  echo "== IFGFB_K4=$k4 (checked build)"
  IFGFB_LIB=$PWD/variants/checked.so IFGFB_K4=$k4 timeout 1200 python -m pytest \
    tests/test_gpu_far.py tests/test_gpu_apply.py tests/test_gpu_partition.py -q -x \
    -k "not slab and not gmres_matches" 2>&1 | tail -3
done
