#!/bin/bash
# round 2 (4m): side-stream placement A/B: hmu inline in stage B; low-priority side stream
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
B="python bench.py --no-dense --serving 0 --no-cpu-baseline"
CAKF_HMU_INLINE=1 timeout 900 $B > gpurun_out/r4m_bench_hmuinline.json 2> gpurun_out/r4m_bench.err
CAKF_SIDE_PRIO=0 timeout 900 $B > gpurun_out/r4m_bench_lowprio.json 2>> gpurun_out/r4m_bench.err
CAKF_HMU_INLINE=1 CAKF_SIDE_PRIO=0 timeout 900 $B > gpurun_out/r4m_bench_both.json 2>> gpurun_out/r4m_bench.err
timeout 900 $B > gpurun_out/r4m_bench.json 2>> gpurun_out/r4m_bench.err
