#!/bin/bash
# round 2 (4k): persistent bulk-copy H M^- side passes (one CTA per SM)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x -k "HM_BULK or STAGE_AB" > gpurun_out/r4k_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r4k_pytest.log
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r4k_bench.json 2> gpurun_out/r4k_bench.err
CAKF_SIDE_PRIO=0 timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r4k_bench_lowprio.json 2>> gpurun_out/r4k_bench.err
