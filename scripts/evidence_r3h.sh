#!/bin/bash
# round 2 (3h): host enqueue vs device time of a cfg3 pass
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python scripts/e2e_breakdown2.py > gpurun_out/r3h_enqueue.json 2> gpurun_out/r3h.err
