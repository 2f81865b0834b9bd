#!/bin/bash
set -x
mkdir -p gpurun_out
python scripts/op_bench.py k2 1 > gpurun_out/op_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gram_gemm_tc_kernel -c 1 -o gpurun_out/prof_k2tc_r1 python scripts/op_bench.py k2 1 > gpurun_out/ncu_k2tc.log 2>&1
echo rc=$?
cat gpurun_out/op_plain.log
