#!/bin/bash
# round 2q: kd order v2 (float4 payload) tests + steady-state launch list (cfg3 steps 40-41 + smoother)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2q_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r2q_pytest.log
timeout 600 python scripts/launch_list_steady.py > gpurun_out/r2q_steady_plain.log 2>&1 && \
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2q_steady.csv python scripts/launch_list_steady.py > gpurun_out/r2q_steady_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2q_steady_ncu.log
