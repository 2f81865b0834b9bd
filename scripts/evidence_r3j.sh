#!/bin/bash
# round 2 (3j): cfg5 sweep re-measured on a dedicated stream (events bracket the library's work)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
rm -f gpurun_out/r3j_cfg5_sweep.jsonl
timeout 3300 python scripts/sweep_cfg5.py --out gpurun_out/r3j_cfg5_sweep.jsonl > gpurun_out/r3j_sweep.log 2>&1
echo "rc=$?" >> gpurun_out/r3j_sweep.log
