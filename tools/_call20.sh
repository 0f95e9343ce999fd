bash tools/ab_variants.sh 4 > gpurun_out/r1s3_ab7.txt 2>&1
bash tools/ab_variants.sh 8 >> gpurun_out/r1s3_ab7.txt 2>&1
echo done
