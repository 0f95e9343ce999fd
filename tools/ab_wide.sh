#!/bin/bash
# A/B of the wide-warp K4 (IFGFB_K4=wide): library variants in variants/*.so x cut
# objectives, at bench size n_refine $1.  usage: tools/ab_wide.sh 4 "2,1,6 1,0,6"
n=${1:-4}
objs=${2:-"2,1,6"}
for lib in variants/*.so; do
  for o in $objs; do
    IFS=, read tw bw r <<< "$o"
    IFGFB_K4=wide IFGFB_WIDE_TW=$tw IFGFB_WIDE_BW=$bw IFGFB_WIDE_CUT=$r IFGFB_LIB=$PWD/$lib \
      python bench.py --n-refine $n --steps 10 --warmup 3 --no-cpu-baseline --no-gmres \
      > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$lib $o FAILED"; tail -3 gpurun_out/ab.err; continue; }
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']; k=d['kernels']
print('%-24s %-8s ms %.3f prop %.3f  %.2f TF frac %.3f' % ('$lib', '$o', d['ms_per_step'], k['propagate']['ms_per_step'], r['achieved'], r['frac']))"
  done
done
