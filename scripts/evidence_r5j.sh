#!/bin/bash
# round 2 (5j): closing bench line (full) and smoke of the final tree
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5j_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/r5j_smoke.log
timeout 900 python bench.py > gpurun_out/r5j_bench.json 2> gpurun_out/r5j_bench.err
timeout 1200 python scripts/parity_table.py --out gpurun_out/r5j_parity_table.json > gpurun_out/r5j_parity.log 2>&1
