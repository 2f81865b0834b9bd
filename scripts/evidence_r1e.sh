#!/bin/bash
# Round-1e evidence: GPU tests, bench line (cfg3 defaults), oracle reference arm, T=3 launch list, K1 full capture.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1e.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_r1e.log
timeout 900 python bench.py > gpurun_out/bench_r1e.json 2> gpurun_out/bench_r1e.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_r1e.json 2> gpurun_out/bench_ref_r1e.err; echo "ref rc=$?"
CMD="python bench.py --config cfg3 --T 3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-dense --no-interp"
$CMD > gpurun_out/plain_t3.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r1e_t3.csv $CMD > gpurun_out/ncu_list_r1e.log 2>&1; echo "list rc=$?"
CMD="python bench.py --config cfg3 --T 10 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-dense --no-interp"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"matvec_sym_kernel" --launch-skip 500 \
  --launch-count 1 -o gpurun_out/prof_k1_r1e $CMD > gpurun_out/ncu_k1_r1e.log 2>&1; echo "k1 rc=$?"
