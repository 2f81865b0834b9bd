#!/bin/bash
# round 2p: own kd order (no CUB) + device-side observation cache: GPU tests, bench, T=3 launch list
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2p_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r2p_pytest.log
timeout 900 python bench.py > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err
CMD="python bench.py --config cfg3 --T 3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-dense --no-interp --serving 0"
timeout 600 $CMD > gpurun_out/r2p_plain_t3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2p_launches_t3.csv $CMD > gpurun_out/r2p_ncu_list.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2p_ncu_list.log
