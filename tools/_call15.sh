timeout 900 python -m pytest tests/test_gpu_apply.py -x -q -k "sl1 or slab" > gpurun_out/r1s3_sl1_tests.log 2>&1
bash tools/ab_variants.sh 4 > gpurun_out/r1s3_ab4.txt 2>&1
echo done
