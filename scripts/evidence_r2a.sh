#!/bin/bash
# round 2a: GPU tests (incl. new parity tests), parity table, bench line.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -s > gpurun_out/r2a_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r2a_pytest.log
timeout 900 python scripts/parity_table.py --out gpurun_out/r2a_parity_table.json > gpurun_out/r2a_parity.log 2>&1; echo "parity_rc=$?" >> gpurun_out/r2a_parity.log
timeout 900 python bench.py --no-dense --no-interp --serving 0 --no-cpu-baseline > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench_rc=$?" >> gpurun_out/r2a_bench.err
tail -3 gpurun_out/r2a_pytest.log
