CMD="python bench.py --config cfg3 --T 3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-dense --no-interp"
$CMD > gpurun_out/plain_t3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv $CMD > gpurun_out/ncu_list_b.log 2>&1
echo "ncu rc=$?"
