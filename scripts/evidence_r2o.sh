#!/bin/bash
# round 2o: full GPU suite (incl. blockres, multi-GPU emulation tests), parity table, cfg3 bench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/r2o_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r2o_pytest.log
timeout 1200 python scripts/parity_table.py --out gpurun_out/r2o_parity_table.json > gpurun_out/r2o_parity.log 2>&1
timeout 900 python bench.py > gpurun_out/r2o_bench.json 2> gpurun_out/r2o_bench.err
