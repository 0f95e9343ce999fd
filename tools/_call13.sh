S="python tools/solve.py --geometry slab --n-refine 1 --max-iter 40 --tol 1e-12"
$S --incident plane-y > gpurun_out/h1.json 2>/dev/null
$S --eps-r 2.25 > gpurun_out/h2.json 2>/dev/null
$S --eps-r 2.25 --incident plane-y > gpurun_out/h3.json 2>/dev/null
bash tools/ab_variants.sh 4 > gpurun_out/r1s3_ab3.txt 2>&1
IFGFB_OVERLAP_EMIT=0 IFGFB_LIB=$PWD/variants/b_pf12.so python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-gmres > gpurun_out/ab_noov.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab_noov.json')); print('no-overlap pf12 ms', d['ms_per_step'], {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" >> gpurun_out/r1s3_ab3.txt
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r1s3_gpu_tests5.log 2>&1
echo done
