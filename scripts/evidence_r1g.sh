#!/bin/bash
# Round-1g evidence: GPU tests, smoke, bench line (cfg3 defaults), oracle reference arm, torchrun N=1 launch check,
# T=3 launch list, one full K1 capture.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1g.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_r1g.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1g.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_r1g.json 2> gpurun_out/bench_r1g.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_r1g.json 2> gpurun_out/bench_ref_r1g.err; echo "ref rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 1 --warmup 3 --no-dense --no-interp --no-cpu-baseline > gpurun_out/bench_torchrun_r1g.json \
  2> gpurun_out/bench_torchrun_r1g.err; echo "torchrun rc=$?"
CMD="python bench.py --config cfg3 --T 3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-dense --no-interp"
$CMD > gpurun_out/plain_t3.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r1g_t3.csv $CMD > gpurun_out/ncu_list_r1g.log 2>&1; echo "list rc=$?"
CMD="python bench.py --config cfg3 --T 10 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-dense --no-interp"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"matvec_sym_kernel" --launch-skip 500 \
  --launch-count 1 -o gpurun_out/prof_k1_r1g $CMD > gpurun_out/ncu_k1_r1g.log 2>&1; echo "k1 rc=$?"
