timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1s3_gpu_final.log 2>&1; echo "exit=$?" >> gpurun_out/r1s3_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1s3_smoke_final.log 2>&1
timeout 900 python bench.py > gpurun_out/r1s3_bench_final.json 2> gpurun_out/r1s3_bench_final.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01_v5_n4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-gmres > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:accum_kernel -s 3 -c 3 -o gpurun_out/ncu_acc_v5 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-gmres > gpurun_out/ncu_acc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"leaf_kernel|emit_kernel|near_kernel" -s 5 -c 3 -o gpurun_out/ncu_other_v5 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-gmres > gpurun_out/ncu_other.log 2>&1
timeout 2700 python tools/solve.py --n-refine 45 --k0-pi 32 --max-iter 50 --tol 1e-12 --device-moments > gpurun_out/r1s3_solve_cfg5_fixed.json 2> gpurun_out/r1s3_solve_cfg5_fixed.err
echo done
