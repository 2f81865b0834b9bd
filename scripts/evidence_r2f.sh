#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
EIG_ONLY=576 EIG_REPS=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:sytrd -c 1 -o gpurun_out/r2f_sytrd python scripts/eig_timing.py > gpurun_out/r2f_ncu.log 2>&1
