#!/bin/bash
# Round-1c evidence: ncu launch list of a T=12 cfg3 pass (ranks reach 512 + 64: truncation, INT8 Gram,
# smoother GEMMs all appear) and one full capture of the INT8-slice GEMM (truncation Gram F^T F).
mkdir -p gpurun_out
CMD="python bench.py --config cfg3 --T 12 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-dense --no-interp"
$CMD > gpurun_out/plain_t12.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1c.csv $CMD \
    > gpurun_out/ncu_list_c.log 2>&1
echo "list rc=$?"
$CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gemm_i8_kernel" --launch-skip 20 --launch-count 1 \
    -o gpurun_out/prof_gemm_i8 $CMD > gpurun_out/ncu_i8.log 2>&1
echo "i8 rc=$?"
