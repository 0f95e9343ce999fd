#!/bin/bash
# A/B the library variants in variants/*.so on the bench workload (n_refine $1):
# c1 parity against the reference golden, then device timing
for lib in variants/*.so; do
  IFGFB_LIB=$PWD/$lib python tools/check_apply.py c1 2>&1 | grep -o "apply rel [0-9.e+-]*" | sed "s|^|$lib |"
  IFGFB_LIB=$PWD/$lib python bench.py --n-refine ${1:-4} --steps 10 --warmup 3 --no-cpu-baseline --no-gmres > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$lib FAILED"; tail -3 gpurun_out/ab.err; continue; }
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']; k=d['kernels']
print('%-28s ms %.3f prop %.3f leaf %.3f emit %.3f near %.3f ms %.2f TF frac %.3f' % ('$lib', d['ms_per_step'], k['propagate']['ms_per_step'], k['leaf']['ms_per_step'], k.get('emit', {}).get('ms_per_step', 0.0), k['near']['ms_per_step'], r['achieved'], r['frac']))"
done
