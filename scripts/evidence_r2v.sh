#!/bin/bash
# round 2v: persistent double-buffered 3xBF16 GEMM (truncation F Q_r): equivalence test, bench; S2 INT8 ncu
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc_persist.py tests/test_gpu_cfg2.py -q -x > gpurun_out/r2v_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r2v_pytest.log
timeout 900 python bench.py --no-dense --serving 0 > gpurun_out/r2v_bench.json 2> gpurun_out/r2v_bench.err
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gemm_i8_kernel -s 0 -c 1 \
  -o gpurun_out/r2v_i8_s2 python scripts/lowrank_bench.py > gpurun_out/r2v_ncu_s2.log 2>&1
echo done >> gpurun_out/r2v_ncu_s2.log
