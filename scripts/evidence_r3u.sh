#!/bin/bash
# round 2 (3u): 16-byte-store bf16x3 transpose-split (truncation), deeper RC-split load unroll
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_lowrank_gemm.py tests/test_gpu_parity.py -q -x > gpurun_out/r3u_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r3u_pytest.log
timeout 600 python scripts/lowrank_bench.py > gpurun_out/r3u_lowrank.log 2>&1
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r3u_bench.json 2> gpurun_out/r3u_bench.err
