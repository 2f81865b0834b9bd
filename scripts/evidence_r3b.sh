#!/bin/bash
# round 2 (3b): K2 with 16 producer warps + 3/3 stages; one-pass RC slicing; float4 ws_dense / kcar_build
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3b_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r3b_pytest.log
timeout 600 python scripts/lowrank_bench.py > gpurun_out/r3b_lowrank.log 2>&1
timeout 900 python bench.py --no-dense --serving 0 > gpurun_out/r3b_bench.json 2> gpurun_out/r3b_bench.err
