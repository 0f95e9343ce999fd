bash tools/ab_variants.sh 4 > gpurun_out/r1s3_ab6.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1s3_gpu_tests6.log 2>&1
echo done
