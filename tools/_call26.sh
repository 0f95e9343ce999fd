for lib in variants/*.so; do
  IFGFB_LIB=$PWD/$lib python tools/check_apply.py c1 2>&1 | grep -o "apply rel [0-9.e+-]*" | sed "s|^|$lib |"
  IFGFB_LIB=$PWD/$lib python bench.py --geometry slab --n-refine 2 --steps 5 --warmup 3 --no-cpu-baseline --no-gmres > gpurun_out/abs.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/abs.json')); k=d['kernels']
print('$lib slab2 ms %.2f near %.2f prop %.2f' % (d['ms_per_step'], k['near']['ms_per_step'], k['propagate']['ms_per_step']))"
done
