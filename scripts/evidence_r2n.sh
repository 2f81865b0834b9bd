#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for i in 1 2; do timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-interp --no-cpu-baseline > gpurun_out/r2n_bench_cfg2_$i.json 2> gpurun_out/r2n_bench_cfg2_$i.err; echo "rc=$?" >> gpurun_out/r2n_bench_cfg2_$i.err; done
