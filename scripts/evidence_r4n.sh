#!/bin/bash
# round 2 (4n): refreshed full evidence after the K1 sub-tile test rework
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r4n_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r4n_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4n_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/r4n_smoke.log
timeout 1200 python scripts/parity_table.py --out gpurun_out/r4n_parity_table.json > gpurun_out/r4n_parity.log 2>&1
timeout 900 python bench.py > gpurun_out/r4n_bench.json 2> gpurun_out/r4n_bench.err
timeout 600 python scripts/launch_list_steady.py > gpurun_out/r4n_steady_plain.log 2>&1 && \
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r4n_steady.csv python scripts/launch_list_steady.py > gpurun_out/r4n_steady_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r4n_steady_ncu.log
