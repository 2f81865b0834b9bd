#!/bin/bash
# round 2 (4l): hmu walks the tiles in reverse (L2 reuse of hmts' last tiles); side stream off for reference
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
B="python bench.py --no-dense --serving 0 --no-cpu-baseline"
timeout 900 $B > gpurun_out/r4l_bench.json 2> gpurun_out/r4l_bench.err
CAKF_HMU_REV=0 timeout 900 $B > gpurun_out/r4l_bench_norev.json 2>> gpurun_out/r4l_bench.err
CAKF_NO_SIDE_STREAM=1 timeout 900 $B > gpurun_out/r4l_bench_noside.json 2>> gpurun_out/r4l_bench.err
