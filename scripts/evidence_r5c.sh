#!/bin/bash
# round 2 (5c): final evidence after the eigensolver work — full GPU suite, smoke, parity table, cfg3 bench (full line), cfg2 lines,
# cfg4 on one GPU, steady-state launch list, source-level ncu of the steady K1
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r5c_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r5c_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5c_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/r5c_smoke.log
timeout 1200 python scripts/parity_table.py --out gpurun_out/r5c_parity_table.json > gpurun_out/r5c_parity.log 2>&1
timeout 900 python bench.py > gpurun_out/r5c_bench.json 2> gpurun_out/r5c_bench.err
timeout 900 python bench.py --config cfg2 --no-dense > gpurun_out/r5c_bench_cfg2_f32.json 2> gpurun_out/r5c_cfg2_f32.err
timeout 900 python bench.py --config cfg2 --dtype f64 --no-dense --serving 0 > gpurun_out/r5c_bench_cfg2_f64.json 2> gpurun_out/r5c_cfg2_f64.err
timeout 1800 python scripts/run_cfg4.py 20 > gpurun_out/r5c_cfg4.json 2> gpurun_out/r5c_cfg4.err
timeout 600 python scripts/launch_list_steady.py > gpurun_out/r5c_steady_plain.log 2>&1 && \
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r5c_steady.csv python scripts/launch_list_steady.py > gpurun_out/r5c_steady_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r5c_steady_ncu.log
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:matvec_sym -s 5 -c 1 \
  -o gpurun_out/r5c_k1 python scripts/launch_list_steady.py > gpurun_out/r5c_ncu_k1.log 2>&1
echo "rc=$?" >> gpurun_out/r5c_ncu_k1.log
