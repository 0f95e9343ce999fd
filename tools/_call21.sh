IFGFB_OTF_MIN_FRAC=0 timeout 900 python bench.py --n-refine 16 --steps 2 --warmup 3 --no-cpu-baseline --no-gmres > gpurun_out/otf_old_n16.json 2>/dev/null
timeout 900 python bench.py --n-refine 16 --steps 2 --warmup 3 --no-cpu-baseline --no-gmres > gpurun_out/otf_new_n16.json 2>/dev/null
timeout 1500 python bench.py --n-refine 24 --steps 2 --warmup 3 --no-cpu-baseline --no-gmres > gpurun_out/otf_new_n24.json 2>/dev/null
echo done
