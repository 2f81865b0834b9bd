"""Device eigensolver timing (cakf_sym_eig) on truncation-shaped Grams; run under ncu for the
per-kernel split:  ncu --metrics gpu__time_duration.sum --csv python scripts/eig_timing.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08971_b200 import binding  # noqa: E402

rng = np.random.default_rng(0)
sizes = ((576, 512), (320, 256), (1088, 1024))
if os.environ.get("EIG_ONLY"):
    sizes = tuple((c, r) for c, r in sizes if c == int(os.environ["EIG_ONLY"]))
for c, r in sizes:
    F = rng.standard_normal((4 * c, c)) * np.logspace(2, -6, c)[None, :]
    G = F.T @ F
    binding.sym_eig(G, r)
    t0 = time.perf_counter()
    n = int(os.environ.get("EIG_REPS", "3"))
    for _ in range(n):
        binding.sym_eig(G, r)
    if n:
        print(c, r, "ms per call (incl. alloc + copies)", (time.perf_counter() - t0) / n * 1e3)
