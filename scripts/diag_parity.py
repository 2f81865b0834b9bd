"""Per-step parity diagnostics (device vs oracle) for a few workload variants."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import cakf as ocakf
from paper_2405_08971_b200 import CAKF_FILTER, CAKF_SMOOTH, runner
from synth import make_workload

def run(name, dtype, **kw):
    wl = make_workload(name, **kw)
    trans, _ = runner.transitions(wl)
    h = runner.make_handle(wl, dtype)
    runner.run(h, trans, runner.stage_inputs(wl, dtype), smooth=True)
    fm, fv = runner.collect(h, wl.T, CAKF_FILTER)
    sm, sv = runner.collect(h, wl.T, CAKF_SMOOTH)
    ssm, tr, osm = ocakf.run_workload(wl, dtype_round=np.float32 if dtype == "f32" else None)
    print(f"== {name} {dtype} {kw}")
    for k in range(wl.T + 1):
        st = h.get_stats(k)
        e1 = np.max(np.abs(fm[k]-tr[k].m))/max(np.max(np.abs(tr[k].m)),1e-300)
        e2 = np.max(np.abs(fv[k]-tr[k].var)/np.abs(tr[k].var))
        e3 = np.max(np.abs(sm[k]-osm['m'][k]))/max(np.max(np.abs(osm['m'][k])),1e-300)
        e4 = np.max(np.abs(sv[k]-osm['var'][k])/np.abs(osm['var'][k]))
        o = tr[k].upd
        print(f"k={k:2d} fm {e1:.2e} fv {e2:.2e} sm {e3:.2e} sv {e4:.2e} | res {st['res0']:.3e}->{st['res_final']:.3e} "
              f"(oracle {o.res0 if o else 0:.3e}->{o.res_final if o else 0:.3e}) eta_min {st['eta_min']:.2e} rej {st['rejected']}")
    h.destroy()

if __name__ == "__main__":
    run("sphere24", "f64", T=3, max_iter=16, max_rank=24)
    run("sphere24", "f32", T=3, max_iter=16, max_rank=24)
    run("sphere24", "f32", T=3, max_iter=16, max_rank=-1)
    run("sphere24", "f32", T=3, max_iter=4, max_rank=-1)
    run("sphere48", "f32", T=3, max_iter=8, max_rank=-1)
    run("cfg1", "f32", T=50)
