timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1s3_gpu_tests4.log 2>&1
python tools/solve.py --n-refine 12 --k0-pi 12 --max-iter 30 --tol 1e-12 > gpurun_out/f1.json 2>/dev/null
python tools/solve.py --geometry slab --n-refine 2 --tol 1e-5 --max-iter 300 > gpurun_out/f2.json 2>/dev/null
echo done
