#!/bin/bash
# round 2 (3c): source-level ncu of the steady-state K1 (cfg3 step 40) for the stall map
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:matvec_sym -s 5 -c 1 \
  -o gpurun_out/r3c_k1 python scripts/launch_list_steady.py > gpurun_out/r3c_ncu_k1.log 2>&1
echo "rc=$?" >> gpurun_out/r3c_ncu_k1.log
