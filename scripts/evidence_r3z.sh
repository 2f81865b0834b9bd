#!/bin/bash
# round 2 (3z): ncu --set full of the stacked INT8 GEMM at S2 (D x 513 x 512)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_i8_kernel -s 0 -c 1 \
  -o gpurun_out/r3z_i8_s2 python scripts/lowrank_bench.py > gpurun_out/r3z_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r3z_ncu.log
