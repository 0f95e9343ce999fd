#!/bin/bash
# Per-rank share of an R-way multi-GPU matvec, measured on ONE GPU: each
# rank's plan (its level-3 window + target rows, built exactly as that rank
# process builds it) is created and timed in its own process, one after
# another (nothing waits on another rank; no collective).  Output: one JSON
# line per rank (bench.py --emulate-ranks) -> max-over-ranks projection.
#   bash tools/rank_sweep.sh 8 "--n-refine 45 --k0-pi 32" > gpurun_out/ranks.jsonl
R=${1:-8}
ARGS=${2:-}
for ((r = 0; r < R; r++)); do
  timeout 1200 python bench.py $ARGS --emulate-ranks $R --emulate-rank $r --steps 5 --warmup 3 \
    --no-cpu-baseline --no-gmres 2> gpurun_out/rank_$r.err || tail -3 gpurun_out/rank_$r.err
done
