#!/bin/bash
# Full ncu capture of one symmetric K1 launch (culled, packed f32x2) at filter step 8 of cfg3.
CMD="python bench.py --config cfg3 --T 10 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"matvec_sym_kernel" --launch-skip 500 --launch-count 1 \
    -o gpurun_out/prof_k1_sym $CMD > gpurun_out/ncu_k1.log 2>&1
echo "rc=$?"
