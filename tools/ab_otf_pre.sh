#!/bin/bash
# A/B of the node-table pre-pass on on-device-geometry levels (every level forced on-device):
# usage: tools/ab_otf_pre.sh [n_refine]
n=${1:-8}
for cfg in "tables IFGFB_GEOM_ON_DEVICE=none" "inkernel IFGFB_GEOM_ON_DEVICE=all IFGFB_OTF_PRE_MB=0" "prepass IFGFB_GEOM_ON_DEVICE=all" "prepass_256MB IFGFB_GEOM_ON_DEVICE=all IFGFB_OTF_PRE_MB=256"; do
  set -- $cfg; name=$1; shift
  env "$@" python bench.py --n-refine $n --steps 10 --warmup 3 --no-cpu-baseline --no-gmres > gpurun_out/ab_otf_$name.json 2> gpurun_out/ab_otf_$name.err || tail -5 gpurun_out/ab_otf_$name.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_otf_$name.json')); r=d['roofline']
print('$name n=$n: ms %.3f  K4 %.3f ms %.2f TF frac %.3f launches %d plan_gib %s' % (d['ms_per_step'], d['kernels']['propagate']['ms_per_step'], r['achieved'], r['frac'], d['gpu_launches'], d['config'].get('device_plan_gib')))"
done
