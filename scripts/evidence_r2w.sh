#!/bin/bash
# round 2w: ncu --set full of the steady-state K = 64 strip GEMM (smoother) and the post-loop K2 (filter)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:gemm_f64acc_strip -c 1 \
  -o gpurun_out/r2w_strip python scripts/launch_list_steady.py > gpurun_out/r2w_ncu_strip.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:gram_gemm_tc -c 1 \
  -o gpurun_out/r2w_k2 python scripts/launch_list_steady.py > gpurun_out/r2w_ncu_k2.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:mix4_kernel -s 3 -c 1 \
  -o gpurun_out/r2w_mix4 python scripts/launch_list_steady.py > gpurun_out/r2w_ncu_mix4.log 2>&1
echo done >> gpurun_out/r2w_ncu_mix4.log
