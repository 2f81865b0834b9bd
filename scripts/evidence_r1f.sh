#!/bin/bash
# Round-1e evidence: GPU tests, bench line (cfg3 defaults), oracle reference arm, T=3 launch list, K1 full capture.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1f.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_r1f.log
timeout 900 python bench.py > gpurun_out/bench_r1f.json 2> gpurun_out/bench_r1f.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_r1f.json 2> gpurun_out/bench_ref_r1f.err; echo "ref rc=$?"
CMD="python bench.py --config cfg3 --T 3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-dense --no-interp"
$CMD > gpurun_out/plain_t3.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r1f_t3.csv $CMD > gpurun_out/ncu_list_r1f.log 2>&1; echo "list rc=$?"
