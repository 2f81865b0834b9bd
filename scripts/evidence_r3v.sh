#!/bin/bash
# round 2 (3v): float4 loads in the one-pass K-contiguous INT8 slicing
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lowrank_gemm.py tests/test_gpu_cfg2.py -q -x > gpurun_out/r3v_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r3v_pytest.log
timeout 600 python scripts/lowrank_bench.py > gpurun_out/r3v_lowrank.log 2>&1
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r3v_bench.json 2> gpurun_out/r3v_bench.err
