#!/bin/bash
# round 2 (5m): dots pass with three row pairs per lane in flight (owner warp separate)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CAKF_LIB=paper_2405_08971_b200/libcakf_trdtiming.so EIG_ONLY=576 EIG_REPS=1 timeout 600 python scripts/eig_timing.py > gpurun_out/r5m_trd_cycles.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "eig or parity or trunc" > gpurun_out/r5m_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r5m_pytest.log
B="python bench.py --no-dense --serving 0 --no-cpu-baseline"
timeout 900 $B > gpurun_out/r5m_bench.json 2> gpurun_out/r5m_bench.err
