#!/bin/bash
# Round-1 evidence: official bench line (cfg3, N=1, defaults), the oracle reference arm, and an ncu
# launch list of a T=3 run of the same path (per-launch durations, cold-cache, serialised).
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_r1.json 2> gpurun_out/bench_ref_r1.err
echo "ref rc=$?"
CMD="python bench.py --config cfg3 --T 3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-dense --no-interp"
$CMD > gpurun_out/plain_t3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv $CMD > gpurun_out/ncu_list_b.log 2>&1
echo "ncu rc=$?"
