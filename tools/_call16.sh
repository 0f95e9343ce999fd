bash tools/ab_variants.sh 4 > gpurun_out/r1s3_ab5.txt 2>&1
echo done
