#!/bin/bash
# round 2 (4i): K1 warps skip row tiles without an active sub-tile; source-level ncu of the steady K1
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "gram or fullsize or k1 or parity" > gpurun_out/r4i_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r4i_pytest.log
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r4i_bench.json 2> gpurun_out/r4i_bench.err
timeout 900 python bench.py --no-dense --serving 0 --no-cpu-baseline > gpurun_out/r4i_bench2.json 2>> gpurun_out/r4i_bench.err
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:matvec_sym -s 5 -c 1 \
  -o gpurun_out/r4i_k1 python scripts/launch_list_steady.py > gpurun_out/r4i_ncu_k1.log 2>&1
echo "rc=$?" >> gpurun_out/r4i_ncu_k1.log
