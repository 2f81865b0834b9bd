#!/bin/bash
# A/B of env-selected variants on the cfg3 bench (no dense / interp / cpu legs): ab.sh "ENV=.. ENV2=.." ...
mkdir -p gpurun_out
for v in "$@"; do
  env $v python bench.py --no-dense --no-interp --no-cpu-baseline --e2e-steps 0 --serving 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  python - "$v" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
    ph = d["phase_ms_per_step"]
    print(f"{sys.argv[1]:40s} {d['value']:.3f} steps/s  k1 {ph['k1_matvec']:.0f}  stages {ph['loop_stages']:.0f}  k2s {ph.get('k2_smooth', ph.get('smooth_kx', 0)):.0f}  k2p {ph['k2_post']:.0f}  lowrank {ph['lowrank']:.0f}  trunc {ph['truncate']:.0f} eig {ph['trunc_eig']:.0f}  frac {d["roofline"]["frac"]:.3f}  evk1 {d["config"]["evaluated_frac"]["k1_matvec"]:.4f}")
except Exception as e:
    print(sys.argv[1], "FAILED", e); print(open("gpurun_out/ab.err").read()[-2000:])
PY
done
