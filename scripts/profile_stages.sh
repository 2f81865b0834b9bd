#!/bin/bash
# Launch list of one late filter step (rank-in 512) of cfg3: per-kernel durations of the inner loop.
CMD="python bench.py --config cfg3 --T 10 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --launch-skip 4200 --launch-count 600 --log-file gpurun_out/launches_stages.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "rc=$?"
