#!/bin/bash
# round 2 (3o): tridiagonalisation cluster size A/B (16 vs 8 CTAs) at c = 320 / 576 / 1088
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
EIG_REPS=10 timeout 600 python scripts/eig_timing.py > gpurun_out/r3o_eig16.log 2>&1
CAKF_TRD_NC=8 EIG_REPS=10 timeout 600 python scripts/eig_timing.py > gpurun_out/r3o_eig8.log 2>&1
