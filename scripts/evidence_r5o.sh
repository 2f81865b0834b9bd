#!/bin/bash
# round 2 (5o): bench with the sampler timed after a warm-up call
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r5o_bench.json 2> gpurun_out/r5o_bench.err
