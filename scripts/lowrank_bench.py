"""Time the fp32 path's low-rank contraction shapes at cfg3 through cakf_lowrank_gemm (INT8-slice GEMM incl.
its operand slicing; CUDA events around the call).  Shapes (column-major m x n x k, op):
  S2  D x 513 x 512  C -= M Tm       (M-major A: the smoother's M^- (M^-T x) and the filter's M^- U)
  S1  512 x 513 x D  Tm = M^T X      (K = D)
  F2  D x 65 x 512   tmp = M^- U
  G   576 x 576 x D  Gram F^T F
"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_08971_b200 import binding

D = 231360
torch.manual_seed(0)
out = {}
def run(name, ashape, bshape, tb, beta, reps=5):
    """torch row-major A (ashape), B (bshape, transposed if tb): the library computes the transposed
    (column-major) problem, i.e. its A is our B and its m is our n (see binding.lowrank_gemm)"""
    A = torch.randn(ashape, device="cuda")
    B = torch.randn(bshape, device="cuda")
    m, n = ashape[0], (bshape[0] if tb else bshape[1])
    C = torch.randn((m, n), device="cuda")
    binding.lowrank_gemm(A, B, transa=False, transb=tb, alpha=-1.0, beta=beta, C=C)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); binding.lowrank_gemm(A, B, transa=False, transb=tb, alpha=-1.0, beta=beta, C=C); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    out[name] = {"lib_m": n, "lib_n": m, "k": ashape[1], "ms_min": min(ts), "ms_med": sorted(ts)[len(ts) // 2]}
    print(name, out[name], flush=True)
    del A, B, C


run("S2_D_513_512", (513, 512), (512, D), False, 1.0)
run("S1_512_513_D", (513, D), (512, D), True, 0.0)
run("F2_D_65_512", (65, 512), (512, D), False, 0.0)
run("G_576_576_D", (576, D), (576, D), True, 0.0)
print(json.dumps(out))
