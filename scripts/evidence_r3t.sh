#!/bin/bash
# round 2 (3t): grid-wide K1 active-unit list (3 launches instead of one 1-block kernel)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_concurrent.py -q -x > gpurun_out/r3t_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r3t_pytest.log
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r3t_bench.json 2> gpurun_out/r3t_bench.err
