#!/bin/bash
# round 2 (4r): per-phase cycle split of the tridiagonalisation (timing build) and per-kernel eigensolver split
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CAKF_LIB=paper_2405_08971_b200/libcakf_trdtiming.so EIG_ONLY=576 EIG_REPS=1 timeout 600 python scripts/eig_timing.py > gpurun_out/r4r_trd_cycles.log 2>&1
EIG_ONLY=576 EIG_REPS=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4r_eig_kernels.csv python scripts/eig_timing.py > gpurun_out/r4r_eig_ncu.log 2>&1
