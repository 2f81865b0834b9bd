#!/bin/bash
# round 2 (4p): 16-byte loads in stage C (V c, Z c) and the K1 slot sums of stages A / AB
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r4p_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r4p_pytest.log
B="python bench.py --no-dense --serving 0 --no-cpu-baseline"
timeout 900 $B > gpurun_out/r4p_bench.json 2> gpurun_out/r4p_bench.err
timeout 900 $B > gpurun_out/r4p_bench2.json 2>> gpurun_out/r4p_bench.err
