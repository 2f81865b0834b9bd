#!/bin/bash
# round 2 (5q): global-memory tridiagonalisation (c > ~600) back to the fused update + dots pass
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "eig or parity or trunc or cfg4 or fullsize" > gpurun_out/r5q_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r5q_pytest.log
EIG_ONLY=1088 EIG_REPS=5 timeout 600 python scripts/eig_timing.py > gpurun_out/r5q_eig1088.log 2>&1
timeout 1800 python scripts/run_cfg4.py 20 > gpurun_out/r5q_cfg4.json 2> gpurun_out/r5q_cfg4.err
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r5q_bench.json 2> gpurun_out/r5q_bench.err
