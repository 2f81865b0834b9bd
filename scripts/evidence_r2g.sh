#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python bench.py --no-dense --no-interp --serving 0 --no-cpu-baseline > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
EIG_ONLY=576 EIG_REPS=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"bt_apply|dc_gemm|sytrd" -c 12 -o gpurun_out/r2g_eigk python scripts/eig_timing.py > gpurun_out/r2g_ncu.log 2>&1
