#!/bin/bash
# round 2b: device eigensolver tests first, then the full GPU suite and the bench (A/B vs cuSOLVER)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_eig.py -x -q -s > gpurun_out/r2b_eig.log 2>&1; echo "eig_rc=$?" >> gpurun_out/r2b_eig.log
tail -3 gpurun_out/r2b_eig.log
if grep -q "eig_rc=0" gpurun_out/r2b_eig.log; then
  timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/r2b_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r2b_pytest.log
  tail -3 gpurun_out/r2b_pytest.log
  timeout 600 python bench.py --no-dense --no-interp --serving 0 --no-cpu-baseline > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
  CAKF_EIG_CUSOLVER=1 timeout 600 python bench.py --no-dense --no-interp --serving 0 --no-cpu-baseline > gpurun_out/r2b_bench_cusolver.json 2>> gpurun_out/r2b_bench.err
fi
