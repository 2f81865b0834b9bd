"""fp32 accuracy vs the fp64 oracle with trajectory-independent actions (random / coord)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import cakf as ocakf
from paper_2405_08971_b200 import CAKF_FILTER, CAKF_SMOOTH, runner
from synth import make_workload
from synth.workloads import farthest_point_order
EPS = np.finfo(np.float32).eps

def run(name, dtype, **kw):
    wl = make_workload(name, **kw)
    if wl.policy == "coord":
        o = farthest_point_order(wl.coords[wl.obs_idx[0]], wl.max_iter); wl.coord_order = [o.copy() for _ in range(wl.T)]
    trans, _ = runner.transitions(wl)
    h = runner.make_handle(wl, dtype)
    runner.run(h, trans, runner.stage_inputs(wl, dtype), smooth=True)
    fm, fv = runner.collect(h, wl.T, CAKF_FILTER); sm, sv = runner.collect(h, wl.T, CAKF_SMOOTH)
    ssm, tr, osm = ocakf.run_workload(wl, dtype_round=np.float32 if dtype == "f32" else None)
    worst = {}
    for k in range(wl.T + 1):
        sd = np.concatenate([np.full(wl.n_space, ssm.sigma_t(k)[d, d]) for d in range(wl.d_time)])
        for tag, got, ref in (("fm", fm[k], tr[k].m), ("sm", sm[k], osm["m"][k])):
            worst[tag] = max(worst.get(tag, 0), np.max(np.abs(got-ref))/np.max(np.abs(ref)))
        for tag, got, ref in (("fv", fv[k], tr[k].var), ("sv", sv[k], osm["var"][k])):
            worst[tag] = max(worst.get(tag, 0), np.max(np.abs(got-ref)/ref))
            worst[tag+"/eps*Sdd"] = max(worst.get(tag+"/eps*Sdd", 0), np.max(np.abs(got-ref)/(EPS*sd)))
    print(name, dtype, kw, {a: f"{b:.2e}" for a, b in worst.items()})

if __name__ == "__main__":
    for pol in ("random", "coord"):
        run("sphere24", "f32", T=4, max_iter=16, max_rank=24, policy=pol)
        run("sphere24", "f64", T=4, max_iter=16, max_rank=24, policy=pol)
        run("sphere48", "f32", T=4, max_iter=16, max_rank=24, policy=pol)
    run("sphere48", "f32", T=4, max_iter=4, max_rank=8, policy="cg")
    run("sphere24", "f32", T=4, max_iter=16, max_rank=24, policy="random", lam=1.0,
        noise_var=[np.ones(1440)]*4)
