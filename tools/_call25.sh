timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --force-partition --no-cpu-baseline --no-gmres > gpurun_out/r1s3_force_part.json 2> gpurun_out/r1s3_force_part.err
timeout 2400 python bench.py --geometry slab --n-refine 7 --steps 3 --warmup 3 --no-cpu-baseline --no-gmres --device-moments > gpurun_out/r1s3_bench_cfg4_r7.json 2> gpurun_out/r1s3_bench_cfg4_r7.err
echo done
