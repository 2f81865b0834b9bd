#!/bin/bash
# round 2u: INT8 GEMM epilogue software-pipelined; fp64 cfg5 points (is the CG RMSE pattern numerical?)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lowrank_gemm.py -q -x > gpurun_out/r2u_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r2u_pytest.log
timeout 600 python scripts/lowrank_bench.py > gpurun_out/r2u_lowrank.log 2>&1
timeout 1500 python scripts/sweep_cfg5.py --out gpurun_out/r2u_cfg5_f64.jsonl --policies cg --iters 16,32,64 --ranks 512 --dtype f64 > gpurun_out/r2u_sweep.log 2>&1
