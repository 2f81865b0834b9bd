#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
CMD="python bench.py --config cfg3 --T 14 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain_t14.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_t14.csv $CMD > gpurun_out/ncu_t14.log 2>&1
echo "rc=$?"
