#!/bin/bash
# round 2y: A/B of the K = 64 products on the INT8 GEMM (CAKF_I8_MIN_K=64) vs the DMMA strip kernel
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2y_bench_default.json 2> gpurun_out/r2y_default.err
CAKF_I8_MIN_K=64 timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2y_bench_i8k64.json 2> gpurun_out/r2y_i8k64.err
CAKF_I8_MIN_K=64 timeout 900 python -m pytest tests/test_gpu_cfg2.py tests/test_gpu_parity.py -q -x > gpurun_out/r2y_pytest_i8k64.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r2y_pytest_i8k64.log
