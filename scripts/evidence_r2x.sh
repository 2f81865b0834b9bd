#!/bin/bash
# round 2x: INT8 GEMM with 8 epilogue warps; mix4 with 4 quads per thread: full GPU suite, shapes, bench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2x_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r2x_pytest.log
timeout 600 python scripts/lowrank_bench.py > gpurun_out/r2x_lowrank.log 2>&1
timeout 900 python bench.py --no-dense --serving 0 > gpurun_out/r2x_bench.json 2> gpurun_out/r2x_bench.err
