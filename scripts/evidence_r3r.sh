#!/bin/bash
# round 2 (3r): smoother carriers forked after the truncation's Gram (beside the eigensolver only)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_cfg2.py -q -x > gpurun_out/r3r_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r3r_pytest.log
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r3r_bench.json 2> gpurun_out/r3r_bench.err
CAKF_SMOOTH_OVERLAP=0 timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r3r_bench_nooverlap.json 2> gpurun_out/r3r_bench_no.err
