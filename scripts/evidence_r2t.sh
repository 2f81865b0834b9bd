#!/bin/bash
# round 2t: INT8 GEMM epilogue (grouped loads + L2 prefetch of old C during the MMAs)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lowrank_gemm.py tests/test_gpu_cfg2.py -q -x > gpurun_out/r2t_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r2t_pytest.log
timeout 600 python scripts/lowrank_bench.py > gpurun_out/r2t_lowrank.log 2>&1
timeout 900 python bench.py --no-dense --serving 0 > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err
