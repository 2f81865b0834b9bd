#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 120 compute-sanitizer --tool memcheck ./scripts/cluster_sync_bench > gpurun_out/r2d_cluster_sync.txt 2>&1
EIG_ONLY=576 EIG_REPS=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:sytrd -c 1 -o gpurun_out/r2d_sytrd python scripts/eig_timing.py > gpurun_out/r2d_ncu.log 2>&1
EIG_ONLY=576 EIG_REPS=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:backtransform -c 1 -o gpurun_out/r2d_bt python scripts/eig_timing.py >> gpurun_out/r2d_ncu.log 2>&1
