#!/bin/bash
# ncu evidence for round 1: launch list + full captures of K1 (inner-loop matvec) and the smoother K2.
set -x
CMD="python bench.py --config cfg3 --T 2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:matvec_partial_kernel -s 5 -c 1 -o gpurun_out/prof_k1_r1 $CMD > gpurun_out/ncu_k1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gram_gemm_kernel -s 2 -c 1 -o gpurun_out/prof_k2_r1 $CMD > gpurun_out/ncu_k2.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/ncu_k2.log
