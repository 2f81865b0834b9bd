#!/bin/bash
# round 2 (5u): steady-state launch list of the final tree
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python scripts/launch_list_steady.py > gpurun_out/r5u_steady_plain.log 2>&1 && \
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r5u_steady.csv python scripts/launch_list_steady.py > gpurun_out/r5u_steady_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r5u_steady_ncu.log
