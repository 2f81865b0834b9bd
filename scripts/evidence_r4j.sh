#!/bin/bash
# round 2 (4j): H M^- side passes through shared memory by bulk copies (bytes in flight beside K1)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x -k "HM_BULK" > gpurun_out/r4j_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r4j_pytest.log
timeout 900 python -m pytest tests -m gpu -q -x -k "gram or fullsize or k1 or parity" >> gpurun_out/r4j_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r4j_pytest.log
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r4j_bench.json 2> gpurun_out/r4j_bench.err
CAKF_HM_BULK=0 timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r4j_bench_nobulk.json 2>> gpurun_out/r4j_bench.err
