#!/bin/bash
# round 2 (3x): tridiagonalisation: next reflector's norm formed with the column update (one pass, one barrier fewer)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3x_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r3x_pytest.log
EIG_REPS=10 timeout 600 python scripts/eig_timing.py > gpurun_out/r3x_eig.log 2>&1
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r3x_bench.json 2> gpurun_out/r3x_bench.err
