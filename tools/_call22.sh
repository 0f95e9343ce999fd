timeout 2400 python bench.py --n-refine 45 --k0-pi 32 --device-moments --steps 2 --warmup 3 --no-cpu-baseline --no-gmres > gpurun_out/cfg5_new.json 2> gpurun_out/cfg5_new.err
echo done
