#!/bin/bash
# round 2 (3e): cp.async strip kernel (K = N^ products), column j+1 over DSMEM in the tridiagonalisation
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3e_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r3e_pytest.log
timeout 900 python bench.py --no-dense --serving 0 > gpurun_out/r3e_bench.json 2> gpurun_out/r3e_bench.err
