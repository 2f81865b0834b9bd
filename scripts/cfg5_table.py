"""Markdown rows of the DESIGN.md cfg5 table from a sweep_cfg5.py JSONL (and the fp64 CG runs).

    python scripts/cfg5_table.py profiles/r2_cfg5_sweep.jsonl [profiles/r2_cfg5_cg_f64.jsonl]
"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
f64 = {}
if len(sys.argv) > 2:
    for l in open(sys.argv[2]):
        if l.strip():
            d = json.loads(l)
            if d.get("max_rank") == 512:
                f64[(d["policy"], d["max_iter"])] = d["test_rmse_smoother"]
by = {(d["policy"], d["max_iter"], d["max_rank"]): d for d in rows}
for pol in ("cg", "random", "coord"):
    for it in (16, 32, 64, 128, 256):
        cells = []
        for r in (128, 256, 512, 1024):
            d = by.get((pol, it, r))
            cells.append("%.1f" % d["time_steps_per_s"] if d else "—")
        d = by.get((pol, it, 512))
        rm = "%.2f" % d["test_rmse_smoother"] if d else "—"
        if (pol, it) in f64:
            rm += " (fp64 %.2f)" % f64[(pol, it)]
        var = "%.1f" % d["test_mean_var_smoother"] if d else "—"
        print("| %s | %d | %s | %s | %s |" % (pol, it, " | ".join(cells), rm, var))
