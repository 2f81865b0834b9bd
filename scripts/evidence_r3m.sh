#!/bin/bash
# round 2 (3m): stacked INT8 MMAs only for single-chunk products; cfg3 bench + cfg2 lines (fp32, fp64)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lowrank_gemm.py tests/test_gpu_variants.py -q -x > gpurun_out/r3m_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r3m_pytest.log
timeout 600 python scripts/lowrank_bench.py > gpurun_out/r3m_lowrank.log 2>&1
timeout 900 python bench.py > gpurun_out/r3m_bench.json 2> gpurun_out/r3m_bench.err
timeout 900 python bench.py --config cfg2 --no-dense > gpurun_out/r3m_bench_cfg2_f32.json 2> gpurun_out/r3m_cfg2_f32.err
timeout 900 python bench.py --config cfg2 --dtype f64 --no-dense --serving 0 > gpurun_out/r3m_bench_cfg2_f64.json 2> gpurun_out/r3m_cfg2_f64.err
