#!/bin/bash
# A/B of near-field kernel builds (variants/*.so) on a sphere and a slab: near ms per matvec
for lib in variants/*.so; do
  for cfg in "--n-refine 8" "--geometry slab --n-refine 3"; do
    IFGFB_LIB=$PWD/$lib python bench.py $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-gmres 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', '$cfg', 'ms', round(d['ms_per_step'],2), 'near', round(d['kernels']['near']['ms_per_step'],3))"
  done
  IFGFB_LIB=$PWD/$lib python tools/check_apply.py c1 2>&1 | grep -o "apply rel [0-9.e+-]*" | sed "s|^|$lib |"
done
