#!/bin/bash
# scratch size of the node-table pre-pass (every level forced on-device): usage tools/ab_otf_scratch.sh [n_refine]
n=${1:-8}
for cfg in "inst16k IFGFB_OTF_PRE_INST=16384" "inst32k IFGFB_OTF_PRE_INST=32768" "inst64k IFGFB_OTF_PRE_INST=65536" "inst256k IFGFB_OTF_PRE_INST=262144" "mb1024 IFGFB_OTF_PRE_MB=1024" "mb4096 IFGFB_OTF_PRE_MB=4096" "mb16384 IFGFB_OTF_PRE_MB=16384"; do
  set -- $cfg; name=$1; shift
  env IFGFB_GEOM_ON_DEVICE=all "$@" python bench.py --n-refine $n --steps 10 --warmup 3 --no-cpu-baseline --no-gmres > gpurun_out/ab_scr_$name.json 2> gpurun_out/ab_scr_$name.err || tail -5 gpurun_out/ab_scr_$name.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_scr_$name.json')); r=d['roofline']
print('$name n=$n: ms %.3f  K4 %.3f ms %.2f TF frac %.3f launches/step %d plan_gib %s' % (d['ms_per_step'], d['kernels']['propagate']['ms_per_step'], r['achieved'], r['frac'], d['gpu_launches']/10, d['config'].get('device_plan_gib')))"
done
