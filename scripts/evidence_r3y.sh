#!/bin/bash
# round 2 (3y): CTA-pair A multicast in the stacked INT8 GEMM
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_lowrank_gemm.py -q -x > gpurun_out/r3y_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r3y_pytest.log
timeout 300 python scripts/lowrank_bench.py > gpurun_out/r3y_lowrank.log 2>&1
echo "lowrank_rc=$?" >> gpurun_out/r3y_lowrank.log
