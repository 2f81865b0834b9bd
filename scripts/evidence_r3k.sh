#!/bin/bash
# round 2 (3k): stacked-B INT8 MMAs (5 per k-step, double-buffered accumulators) and stacked 3xBF16 K2 MMAs
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3k_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r3k_pytest.log
timeout 600 python scripts/lowrank_bench.py > gpurun_out/r3k_lowrank.log 2>&1
timeout 900 python bench.py --no-dense --serving 0 > gpurun_out/r3k_bench.json 2> gpurun_out/r3k_bench.err
