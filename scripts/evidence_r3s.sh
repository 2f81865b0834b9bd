#!/bin/bash
# round 2 (3s): K = r_in products with 128 <= r_in < 512 on the INT8 GEMM (was the tiled DMMA kernel)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3s_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r3s_pytest.log
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r3s_bench.json 2> gpurun_out/r3s_bench.err
timeout 900 python bench.py --config cfg2 --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r3s_bench_cfg2.json 2> gpurun_out/r3s_cfg2.err
