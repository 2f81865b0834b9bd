#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_eig.py -x -q > gpurun_out/r2h_eig.log 2>&1; echo "eig_rc=$?" >> gpurun_out/r2h_eig.log
CAKF_LIB=$GRAFT_REPO_ROOT/paper_2405_08971_b200/libcakf_trdtiming.so EIG_REPS=1 timeout 300 python scripts/eig_timing.py > gpurun_out/r2h_trd_timing.txt 2>&1
EIG_REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_eig_ncu.csv python scripts/eig_timing.py > gpurun_out/r2h_eig_ncu.log 2>&1
