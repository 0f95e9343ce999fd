bash tools/ab_variants.sh 4 > gpurun_out/r1s3_ab2.txt 2>&1
timeout 1500 python tools/solve.py --geometry slab --n-refine 4 --tol 1e-5 --max-iter 60 > gpurun_out/g1.json 2> gpurun_out/g1.err
echo done
