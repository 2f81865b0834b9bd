#!/bin/bash
# ncu launch list of the steady-state tail of a T=12 cfg3 pass (last filter steps + the smoother): the
# first 6500 launches are skipped (not profiled)
mkdir -p gpurun_out
CMD="python bench.py --config cfg3 --T 12 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-dense --no-interp"
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 6500 --launch-count 2500 --csv \
    --log-file gpurun_out/launches_tail.csv $CMD > gpurun_out/ncu_list_tail.log 2>&1
echo "list rc=$?"
