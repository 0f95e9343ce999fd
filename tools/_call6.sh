bash tools/ab_variants.sh 4 > gpurun_out/r1s3_ab1.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_far.py -x -q -k full_size > gpurun_out/r1s3_fullsize.log 2>&1
S="python tools/solve.py --max-iter 30 --tol 1e-12"
$S --n-refine 8 > gpurun_out/d1.json 2>/dev/null
$S --n-refine 8 --geom-on-device all --stream-parts 3 > gpurun_out/d2.json 2>/dev/null
$S --n-refine 12 --k0-pi 8.533333333 > gpurun_out/d3.json 2>/dev/null
$S --n-refine 12 --k0-pi 8.533333333 --device-moments > gpurun_out/d4.json 2>/dev/null
echo done
