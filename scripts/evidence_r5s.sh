#!/bin/bash
# round 2 (5s): closing check after the global-memory tridiagonalisation fix
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r5s_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r5s_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5s_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/r5s_smoke.log
timeout 900 python bench.py > gpurun_out/r5s_bench.json 2> gpurun_out/r5s_bench.err
