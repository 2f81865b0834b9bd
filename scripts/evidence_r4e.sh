#!/bin/bash
# round 2 (4e): eigensolver T factors on a side stream beside the divide and conquer
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r4e_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r4e_pytest.log
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r4e_bench.json 2> gpurun_out/r4e_bench.err
