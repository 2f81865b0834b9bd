#!/bin/bash
# round 2 (3i): bench on a dedicated stream (events now bracket the library's work); enqueue check
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python scripts/e2e_breakdown2.py > gpurun_out/r3i_enqueue.json 2> gpurun_out/r3i_enqueue.err
timeout 900 python bench.py > gpurun_out/r3i_bench.json 2> gpurun_out/r3i_bench.err
