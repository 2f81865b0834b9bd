#!/bin/bash
# round 2 (3d): K2 producers arrive once per warp (fence per lane, __syncwarp, lane-0 release)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_cfg2.py -q -x > gpurun_out/r3d_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r3d_pytest.log
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r3d_bench.json 2> gpurun_out/r3d_bench.err
