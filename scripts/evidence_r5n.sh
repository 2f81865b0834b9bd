#!/bin/bash
# round 2 (5n): closing check of the final tree — full GPU suite, smoke, cfg3 bench line
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r5n_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r5n_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5n_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/r5n_smoke.log
timeout 900 python bench.py > gpurun_out/r5n_bench.json 2> gpurun_out/r5n_bench.err
