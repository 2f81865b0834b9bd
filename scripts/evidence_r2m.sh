#!/bin/bash
# cfg2 bench lines (fp32, fp64) and the cfg5 sweep
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 --no-interp > gpurun_out/r2m_bench_cfg2_f32.json 2> gpurun_out/r2m_cfg2.err
timeout 900 python bench.py --config cfg2 --dtype f64 --steps 3 --warmup 3 --no-interp --no-cpu-baseline --serving 0 > gpurun_out/r2m_bench_cfg2_f64.json 2>> gpurun_out/r2m_cfg2.err
rm -f gpurun_out/r2_cfg5_sweep.jsonl
timeout 3000 python scripts/sweep_cfg5.py --out gpurun_out/r2_cfg5_sweep.jsonl > gpurun_out/r2m_sweep.log 2>&1
