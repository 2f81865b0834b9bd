#!/bin/bash
# Round-1d evidence: GPU test suite, smoke, official bench line (cfg3, N=1, defaults), oracle reference arm.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1d.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_r1d.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1d.log 2>&1
echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_r1d.json 2> gpurun_out/bench_r1d.err
echo "bench rc=$?"; cat gpurun_out/bench_r1d.json | head -c 600
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_r1d.json 2> gpurun_out/bench_ref_r1d.err
echo "ref rc=$?"
