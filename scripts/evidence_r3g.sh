#!/bin/bash
# round 2 (3g): e2e breakdown (device vs host inputs, read-backs)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python scripts/e2e_breakdown.py > gpurun_out/r3g_e2e.json 2> gpurun_out/r3g_e2e.err
