#!/bin/bash
# round 2r: K1 exponential split (MUFU / FMA pipe), INT8 GEMM epilogue loads batched: tests, shapes, bench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2r_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r2r_pytest.log
timeout 600 python scripts/lowrank_bench.py > gpurun_out/r2r_lowrank.log 2>&1
timeout 900 python bench.py > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err
