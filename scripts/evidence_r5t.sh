#!/bin/bash
# round 2 (5t): full ncu captures of the steady-state stage AB and stage C kernels (slot lists, 16-byte loads)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:stageAB -s 5 -c 1 \
  -o gpurun_out/r5t_stageab python scripts/launch_list_steady.py > gpurun_out/r5t_ncu_ab.log 2>&1
echo "rc=$?" >> gpurun_out/r5t_ncu_ab.log
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:stageC -s 10 -c 1 \
  -o gpurun_out/r5t_stagec python scripts/launch_list_steady.py > gpurun_out/r5t_ncu_c.log 2>&1
echo "rc=$?" >> gpurun_out/r5t_ncu_c.log
