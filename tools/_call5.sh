timeout 2700 python tools/solve.py --n-refine 45 --k0-pi 32 --max-iter 50 --tol 1e-12 --device-moments > gpurun_out/r1s3_solve_cfg5.json 2> gpurun_out/r1s3_solve_cfg5.err
timeout 900 python tools/solve.py --geometry superellipsoid --n-refine 8 --tol 1e-5 --max-iter 1200 > gpurun_out/r1s3_solve_cfg3_full.json 2> gpurun_out/r1s3_solve_cfg3_full.err
echo done
