#!/bin/bash
# round 2k: full GPU suite, bench, cfg3 T=3 launch list (which kernels run: no cuBLAS / cuSOLVER expected)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2k_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r2k_pytest.log
timeout 600 python bench.py --no-dense --no-interp --serving 0 --no-cpu-baseline > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
CMD="python bench.py --config cfg3 --T 3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-dense --no-interp --serving 0"
$CMD > gpurun_out/r2k_plain_t3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2k_launches_t3.csv $CMD > gpurun_out/r2k_ncu_list.log 2>&1
