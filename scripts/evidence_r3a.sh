#!/bin/bash
# round 2 (3a): A/B of the K2 operand split: 3 x BF16 (default) vs 2 x FP16 (CAKF_K2_PREC=f16x2)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CAKF_K2_PREC=f16x2 timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r3a_bench_f16.json 2> gpurun_out/r3a_f16.err
CAKF_K2_PREC=f16x2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cfg2.py tests/test_gpu_fullsize.py -q > gpurun_out/r3a_pytest_f16.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r3a_pytest_f16.log
