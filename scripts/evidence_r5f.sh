#!/bin/bash
# round 2 (5f): hmu4 in 32-thread blocks
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "eig or parity or trunc or variant" > gpurun_out/r5f_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r5f_pytest.log
B="python bench.py --no-dense --serving 0 --no-cpu-baseline"
timeout 900 $B > gpurun_out/r5f_bench.json 2> gpurun_out/r5f_bench.err
timeout 900 $B > gpurun_out/r5f_bench2.json 2>> gpurun_out/r5f_bench.err
