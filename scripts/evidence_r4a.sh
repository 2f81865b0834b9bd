#!/bin/bash
# round 2 (4a): filter truncation eigensolver + M Q_r on their own stream beside the next update's first K1
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r4a_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r4a_pytest.log
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r4a_bench.json 2> gpurun_out/r4a_bench.err
CAKF_TRUNC_OVERLAP=0 timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r4a_bench_nooverlap.json 2> gpurun_out/r4a_bench_no.err
