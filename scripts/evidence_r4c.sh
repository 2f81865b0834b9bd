#!/bin/bash
# round 2 (4c): stage AB sums only the K1 partial slots written by active units
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_cfg2.py -q -x > gpurun_out/r4c_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r4c_pytest.log
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r4c_bench.json 2> gpurun_out/r4c_bench.err
