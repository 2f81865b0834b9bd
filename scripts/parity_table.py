"""Parity error table: the CUDA path through the C-ABI vs the CPU oracle on the same
seeded inputs, per workload / policy / dtype.  Prints one JSON object per case and writes them to
--out (profiles/r2_parity_table.json).  Columns: max relative mean error (max_k ||dm||_inf/||m||_inf),
max elementwise relative variance error, and the minimum device variance, for the filter (f) and
the smoother (s); for fp64 CG the oracle's own sensitivity to a 1-ulp relative perturbation of y.

    python scripts/parity_table.py [--cases cfg2] [--out profiles/r2_parity_table.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import cakf as ocakf  # noqa: E402
from oracle import mfree  # noqa: E402
from paper_2405_08971_b200 import CAKF_FILTER, CAKF_SMOOTH, runner  # noqa: E402
from synth import make_workload  # noqa: E402
from synth.workloads import farthest_point_order  # noqa: E402

EPS32 = float(np.finfo(np.float32).eps)


def device(wl, dtype):
    trans, _ = runner.transitions(wl)
    h = runner.make_handle(wl, dtype)
    runner.run(h, trans, runner.stage_inputs(wl, dtype), smooth=True)
    h.sync()
    fm, fv = runner.collect(h, wl.T, CAKF_FILTER)
    sm, sv = runner.collect(h, wl.T, CAKF_SMOOTH)
    stats = [h.get_stats(k) for k in range(wl.T + 1)]
    h.destroy()
    return fm, fv, sm, sv, stats


def oracle(wl, dtype, dense, perturb=0.0):
    rnd = np.float32 if dtype == "f32" else None
    if dense:
        if perturb:
            wl = _perturbed(wl, perturb)
        ssm, tr, osm = ocakf.run_workload(wl, dtype_round=rnd)
        return ([t.m for t in tr], [t.var for t in tr], osm["m"], osm["var"])
    out = mfree.run_mf(wl, dtype_round=rnd, cache=True, perturb_y=perturb)
    return out["fm"], out["fv"], out["sm"], out["sv"]


def _perturbed(wl, eps):
    import copy
    w2 = copy.copy(wl)
    w2.y = [y * (1.0 + eps) for y in wl.y]
    return w2


def mrel(a, b):
    den, num = float(np.max(np.abs(b))), float(np.max(np.abs(a - b)))
    return num / den if den > 0 else (0.0 if num == 0 else float("inf"))


def errs(dev, ref, sdd=None):
    fm, fv, sm, sv = dev[:4]
    om, ov, osm_, osv = ref
    vrel = lambda a, b: float(np.max(np.abs(a - b) / np.abs(b)))
    T = len(fm) - 1
    return {"f_mean": max(mrel(fm[k], om[k]) for k in range(T + 1)),
            "f_var": max(vrel(fv[k], ov[k]) for k in range(T + 1)),
            "s_mean": max(mrel(sm[k], osm_[k]) for k in range(T + 1)),
            "s_var": max(vrel(sv[k], osv[k]) for k in range(T + 1)),
            "f_var_min": float(min(np.min(v) for v in fv)), "s_var_min": float(min(np.min(v) for v in sv)),
            # downdate-cancellation constant of R20: max |dv| / (eps32 Sigma_dd)
            "c_cancel": None if sdd is None else float(max(np.max(np.abs(a - b) / (EPS32 * sdd))
                                                           for a, b in zip(list(fv) + list(sv), list(ov) + list(osv))))}


def sens(a, b):
    return errs((a[0], a[1], a[2], a[3]), b)


CASES = {
    "cfg1": [("cfg1", {}, "f64", True), ("cfg1", {}, "f32", True), ("cfg1", {"reorth": False}, "f64", True)],
    "sphere48": [("sphere48", dict(policy="cg", max_iter=16, max_rank=24, T=5), d, True) for d in ("f64", "f32")]
    + [("sphere48", dict(policy="random", max_iter=16, max_rank=24, T=5), d, True) for d in ("f64", "f32")]
    + [("sphere48", dict(policy="cg", max_iter=16, max_rank=24, T=5, reorth=False), "f64", True)],
    "sphere24": [("sphere24", dict(policy=p, max_iter=16, max_rank=24, T=4), d, True)
                 for p in ("random", "coord", "cg") for d in ("f64", "f32")],
    "blockres": [("sphere48", dict(policy="blockres", max_iter=16, max_rank=24, T=5, block_actions=4), d, True)
                 for d in ("f64", "f32")],
    "cfg2": [("cfg2", dict(policy=p, T=6), d, False) for p in ("random", "coord", "cg") for d in ("f64", "f32")]
    + [("cfg2", dict(policy="cg", T=6, max_iter=6, max_rank=16), d, False) for d in ("f64", "f32")],
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="cfg1,sphere48,sphere24,blockres,cfg2")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    for group in args.cases.split(","):
        for name, kw, dtype, dense in CASES[group]:
            wl = make_workload(name, **kw)
            if wl.policy == "coord" and name != "cfg1":
                o = farthest_point_order(wl.coords[wl.obs_idx[0]], wl.max_iter)
                wl.coord_order = [o.copy() for _ in range(wl.T)]
            t0 = time.time()
            dev = device(wl, dtype)
            t1 = time.time()
            ref = oracle(wl, dtype, dense)
            sdd = np.concatenate([np.full(wl.n_space, wl.sigma ** 2), np.full(wl.n_space, 3 * wl.sigma ** 2 / wl.ell_t ** 2)])
            row = {"case": name, "dtype": dtype, "policy": wl.policy, "max_iter": wl.max_iter,
                   "max_rank": wl.max_rank, "T": wl.T, "D": wl.D, "reorth": bool(wl.reorth),
                   "oracle": "dense O4/O5" if dense else "matrix-free O8 (cached kernel matrices)",
                   **errs(dev, ref, sdd if dtype == "f32" else None), "ranks_out": [s["rank_out"] for s in dev[4][1:]],
                   "device_s": round(t1 - t0, 2), "oracle_s": round(time.time() - t1, 2)}
            if wl.policy == "cg" and dtype == "f64":
                ref2 = oracle(wl, dtype, dense, perturb=2.0 ** -52)
                row["oracle_1ulp_sensitivity"] = sens(ref2, ref)
            print(json.dumps(row), flush=True)
            rows.append(row)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
