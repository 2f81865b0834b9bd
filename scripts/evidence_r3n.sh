#!/bin/bash
# round 2 (3n): A/B stacked INT8 ntile 96 (one buffer) vs 48 (two buffers) on the single-chunk products
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CAKF_I8_STACK_MAXN=96 timeout 600 python scripts/lowrank_bench.py > gpurun_out/r3n_lowrank96.log 2>&1
timeout 600 python scripts/lowrank_bench.py > gpurun_out/r3n_lowrank48.log 2>&1
