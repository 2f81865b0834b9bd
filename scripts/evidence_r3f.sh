#!/bin/bash
# round 2 (3f): back-transformation W = V^T Z on all threads (row-split partial sums); DSMEM column read reverted
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_eig.py tests/test_gpu_parity.py -q -x > gpurun_out/r3f_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r3f_pytest.log
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r3f_bench.json 2> gpurun_out/r3f_bench.err
