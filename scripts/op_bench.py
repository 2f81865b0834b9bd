"""Time the fused kernel operators (K1 matvec, K2 kernel-GEMM) at cfg3 shapes via the C-ABI op."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2405_08971_b200 import binding
from synth import make_workload

wl = make_workload("cfg3", T=1)
X = torch.tensor(wl.coords.astype(np.float32), device="cuda")
Xt = X[torch.tensor(wl.obs_idx[0], device="cuda")]
which = sys.argv[1] if len(sys.argv) > 1 else "all"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
def timeit(fn):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(reps)]; e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
if which in ("all", "k2"):
    for C, rows, cols in ((1026, X, X), (65, X, Xt)):
        B = torch.randn(cols.shape[0], C, device="cuda")
        ms = timeit(lambda: binding.gram_matmul(rows, cols, B, 1.5, wl.ell_x))
        fl = 2.0 * rows.shape[0] * cols.shape[0] * C
        print(f"K2 M={rows.shape[0]} K={cols.shape[0]} C={C}: {ms:.2f} ms  {fl/ms/1e9:.1f} TFLOP/s (fp32-equivalent)")
if which in ("all", "k1"):
    s = torch.randn(Xt.shape[0], device="cuda")
    Xt2 = Xt.clone()
    ms = timeit(lambda: binding.gram_matmul(Xt, Xt2, s, 1.5, wl.ell_x))
    print(f"K1(op, dense) N={Xt.shape[0]}: {ms:.3f} ms  {Xt.shape[0]**2/ms/1e6:.1f} Gpair/s")
    ms = timeit(lambda: binding.gram_matmul(Xt, Xt, s, 1.5, wl.ell_x))
    n = Xt.shape[0]
    print(f"K1(op, symmetric) N={n}: {ms:.3f} ms  {n*(n+1)/2/ms/1e6:.1f} unique Gpair/s (incl. host staging)")
