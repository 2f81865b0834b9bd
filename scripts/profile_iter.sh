#!/bin/bash
# Launch list (durations + DRAM bytes) of a window of inner iterations at rank-in 512 (filter step ~9 of cfg3).
CMD="python bench.py --config cfg3 --T 10 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-dense --no-interp"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --launch-skip 4400 --launch-count 60 --log-file gpurun_out/launches_iter.csv $CMD > gpurun_out/ncu_iter.log 2>&1
echo "rc=$?"
