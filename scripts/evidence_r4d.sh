#!/bin/bash
# round 2 (4d): cfg4 (D = 1.0M, N = 376,500, r = 1024) on one GPU, T = 20, with the final round-2 build
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1800 python scripts/run_cfg4.py 20 > gpurun_out/r4d_cfg4.json 2> gpurun_out/r4d_cfg4.err
echo "rc=$?" >> gpurun_out/r4d_cfg4.err
