"""Sweep of the device eigensolver over sizes and matrix structures (diagnostic)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08971_b200 import binding  # noqa: E402

rng = np.random.default_rng(0)
bad = 0
for c in [576, 16, 18, 40, 16, 18, 333, 17] + list(range(2, 80)) + [100, 128, 129, 200, 320, 576]:
    for kind in ("rand", "gram", "lowrank"):
        if kind == "rand":
            A = rng.standard_normal((c, c)); G = A + A.T
        elif kind == "gram":
            F = rng.standard_normal((3 * c, c)) * np.logspace(0, -5, c); G = F.T @ F
        else:
            F = rng.standard_normal((c, max(1, c // 3))); G = F @ F.T
        r = max(1, c - 6) if c % 2 else c
        w, Q = binding.sym_eig(G, r)
        wr = np.linalg.eigvalsh(G)
        sc = np.max(np.abs(wr))
        ew = np.max(np.abs(w - wr)) / sc
        res = np.max(np.linalg.norm(G @ Q - Q * w[::-1][:r], axis=0)) / sc
        orth = np.max(np.abs(Q.T @ Q - np.eye(r)))
        if ew > 1e-12 or res > 1e-11 or orth > 1e-12:
            bad += 1
            print("BAD", c, kind, ew, res, orth)
# the Grams of an actual run (sphere48, T=3, 8 actions, r=10)
from oracle import cakf as ocakf  # noqa: E402
from synth import make_workload  # noqa: E402
wl = make_workload("sphere48", T=3, max_iter=8, max_rank=10)
ssm, tr, _ = ocakf.run_workload(wl, smoother=False)
for k in (2, 3):
    G = tr[k].M.T @ tr[k].M
    w, Q = binding.sym_eig(G, 10)
    wr = np.linalg.eigvalsh(G)
    res = np.max(np.linalg.norm(G @ Q - Q * w[::-1][:10], axis=0)) / np.max(wr)
    print("run gram k", k, G.shape, np.max(np.abs(w - wr)) / np.max(wr), "res", res, "orth", np.max(np.abs(Q.T @ Q - np.eye(10))))
print("bad", bad)
