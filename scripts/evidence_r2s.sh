#!/bin/bash
# round 2s: ncu --set full of the INT8 GEMM at the smoother's S2 shape (D x 513 x 512, M-major A) and K = D (S1)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python scripts/lowrank_bench.py > gpurun_out/r2s_lowrank.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gemm_i8_kernel -s 0 -c 1 \
  -o gpurun_out/r2s_i8_s2 python scripts/lowrank_bench.py > gpurun_out/r2s_ncu_s2.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gemm_i8_kernel -s 6 -c 1 \
  -o gpurun_out/r2s_i8_s1 python scripts/lowrank_bench.py > gpurun_out/r2s_ncu_s1.log 2>&1
echo done >> gpurun_out/r2s_ncu_s1.log
