#!/bin/bash
# round 2 (5r): cfg5 sweep, rank cap 1024 column, after the global-memory tridiagonalisation fix
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python scripts/sweep_cfg5.py --out gpurun_out/r5r_cfg5_r1024.jsonl --ranks 1024 > gpurun_out/r5r_sweep.log 2>&1
echo "rc=$?" >> gpurun_out/r5r_sweep.log
