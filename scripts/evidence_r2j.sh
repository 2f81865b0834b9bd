#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CAKF_EIG_CHECK=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "predictive_moments" > gpurun_out/r2j_check.txt 2>&1
CAKF_EIG_CUSOLVER=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "predictive_moments or sphere48_fp64" >> gpurun_out/r2j_check.txt 2>&1
