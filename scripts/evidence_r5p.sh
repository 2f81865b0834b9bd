#!/bin/bash
# round 2 (5p): cfg5 sweep re-measured on the final tree
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 3000 python scripts/sweep_cfg5.py --out gpurun_out/r5p_cfg5_sweep.jsonl > gpurun_out/r5p_sweep.log 2>&1
echo "rc=$?" >> gpurun_out/r5p_sweep.log
