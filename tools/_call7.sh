S="python tools/solve.py --max-iter 20 --tol 1e-12"
$S --n-refine 4 > gpurun_out/e1.json 2>/dev/null
$S --n-refine 4 --k0-pi 2.8444444444 > gpurun_out/e2.json 2>/dev/null
$S --n-refine 6 --k0-pi 4.2666666667 > gpurun_out/e3.json 2>/dev/null
$S --n-refine 12 --k0-pi 12 > gpurun_out/e4.json 2>/dev/null
$S --n-refine 4 --k0-pi 3.5 > gpurun_out/e5.json 2>/dev/null
echo done
