#!/bin/bash
# usage: tools/quick_perf.sh [n_refine]  -- parity at c1 + device timing at the bench size
python tools/check_apply.py c1 2>&1 | grep -E "apply rel|device apply"
python bench.py --n-refine ${1:-4} --steps 10 --warmup 3 --no-cpu-baseline --no-gmres > gpurun_out/qp.json 2> gpurun_out/qp.err || tail -5 gpurun_out/qp.err
python -c "
import json; d=json.load(open('gpurun_out/qp.json')); r=d['roofline']
print('value %.4g  ms %.3f  prop %.2f TF frac %.3f' % (d['value'], d['ms_per_step'], r['achieved'], r['frac']))
print({k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
