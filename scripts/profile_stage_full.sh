#!/bin/bash
# Full ncu capture of the inner-loop stage kernels at rank-in 512 (filter step 9 of cfg3).
CMD="python bench.py --config cfg3 --T 10 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stage[ABC]_kernel|matvec_sym_kernel" --launch-skip 2600 --launch-count 5 \
    -o gpurun_out/prof_stages $CMD > gpurun_out/ncu_stages.log 2>&1
echo "rc=$?"
