#!/bin/bash
# round 2 (5v): hmu launched with programmatic dependent launch after hmts
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r5v_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r5v_pytest.log
B="python bench.py --no-dense --serving 0 --no-cpu-baseline"
timeout 900 $B > gpurun_out/r5v_bench.json 2> gpurun_out/r5v_bench.err
timeout 900 $B > gpurun_out/r5v_bench2.json 2>> gpurun_out/r5v_bench.err
