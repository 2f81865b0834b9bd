#!/bin/bash
# Full ncu capture of one smoother K2 launch (gram_gemm_tc_kernel, culled) at cfg3.
CMD="python bench.py --config cfg3 --T 12 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-dense --no-interp"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_k2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gram_gemm_tc_kernel" --launch-skip 16 --launch-count 1 \
    -o gpurun_out/prof_k2_tc $CMD > gpurun_out/ncu_k2.log 2>&1
echo "rc=$?"
