#!/bin/bash
# round 2 (5i): stage kernels sum only the K1 partial slots that can be nonzero (per-block partner lists)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r5i_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r5i_pytest.log
B="python bench.py --no-dense --serving 0 --no-cpu-baseline"
timeout 900 $B > gpurun_out/r5i_bench.json 2> gpurun_out/r5i_bench.err
CAKF_SLOT_LISTS=0 timeout 900 $B > gpurun_out/r5i_bench_nolists.json 2>> gpurun_out/r5i_bench.err
timeout 900 $B > gpurun_out/r5i_bench2.json 2>> gpurun_out/r5i_bench.err
