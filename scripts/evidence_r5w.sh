#!/bin/bash
# round 2 (5w): cfg2 bench lines on the final tree
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg2 --no-dense > gpurun_out/r5w_bench_cfg2_f32.json 2> gpurun_out/r5w_cfg2_f32.err
timeout 900 python bench.py --config cfg2 --dtype f64 --no-dense --serving 0 > gpurun_out/r5w_bench_cfg2_f64.json 2> gpurun_out/r5w_cfg2_f64.err
