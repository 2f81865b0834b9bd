#!/bin/bash
# round 2 (4h): K1 sub-tile test lane-parallel (one ballot per row tile), squared compares, + bounding boxes
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "gram or fullsize or k1 or parity" > gpurun_out/r4h_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r4h_pytest.log
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r4h_bench.json 2> gpurun_out/r4h_bench.err
CAKF_K1_BOX=0 timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r4h_bench_nobox.json 2>> gpurun_out/r4h_bench.err
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r4h_bench2.json 2>> gpurun_out/r4h_bench.err
