#!/bin/bash
# round 2 (4u): K1 partial sub-tile path two sub-tiles at a time
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "gram or fullsize or k1 or parity" > gpurun_out/r4u_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r4u_pytest.log
B="python bench.py --no-dense --serving 0 --no-cpu-baseline"
timeout 900 $B > gpurun_out/r4u_bench.json 2> gpurun_out/r4u_bench.err
timeout 900 $B > gpurun_out/r4u_bench2.json 2>> gpurun_out/r4u_bench.err
