#!/bin/bash
# ncu launch list of a T=12 cfg3 pass (ranks reach 512 + 64 from step 9: every kernel of the steady state appears)
mkdir -p gpurun_out
CMD="python bench.py --config cfg3 --T 12 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-dense --no-interp"
$CMD > gpurun_out/plain_t12.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_t12.csv $CMD \
    > gpurun_out/ncu_list_t12.log 2>&1
echo "list rc=$?"
