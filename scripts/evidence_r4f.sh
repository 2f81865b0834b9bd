#!/bin/bash
# round 2 (4f): K1 row groups rotate with the row tile (evens out culled work per warp)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "gram or fullsize or k1 or parity" > gpurun_out/r4f_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r4f_pytest.log
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r4f_bench.json 2> gpurun_out/r4f_bench.err
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r4f_bench2.json 2>> gpurun_out/r4f_bench.err
