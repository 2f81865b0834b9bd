"""Time the INT8-slice GEMM (cakf_lowrank_gemm) on the cfg3 low-rank shapes against cuBLAS DGEMM
on fp64 copies (what the fp32 path used before).  CUDA events, after warm-up.

    python scripts/gemm_i8_bench.py [--reps 5]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08971_b200 import binding  # noqa: E402

D, R, C, NHAT, N = 231360, 512, 513, 64, 87120
# (name, m, n, k, transa, transb): C(m x n) = op(A) op(B)
SHAPES = [
    ("gram F^T F", 576, 576, D, True, False),
    ("M Q_r", D, 512, 576, False, False),
    ("smoother M^T x", R, C, D, True, False),
    ("smoother M (M^T x)", D, C, R, False, False),
    ("smoother B_k t", D, C, NHAT, False, False),
    ("post HM^T [v V]", R, NHAT + 1, N, True, False),
    ("post M U", D, NHAT + 1, R, False, False),
]


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    out = []
    for name, m, n, k, ta, tb in SHAPES:
        if args.only and args.only not in name:
            continue
        A = torch.randn((k, m) if ta else (m, k), device="cuda", generator=g)
        B = torch.randn((n, k) if tb else (k, n), device="cuda", generator=g)
        Ad, Bd = A.double(), B.double()
        opA = (lambda: Ad.t()) if ta else (lambda: Ad)
        opB = (lambda: Bd.t()) if tb else (lambda: Bd)
        t_i8 = timed(lambda: binding.lowrank_gemm(A, B, transa=ta, transb=tb), args.reps)
        t_d = timed(lambda: opA() @ opB(), args.reps)
        t_cv = timed(lambda: (A.double(), B.double()), args.reps)
        rec = {"shape": name, "m": m, "n": n, "k": k, "i8_ms": round(t_i8, 3), "dgemm_ms": round(t_d, 3),
               "convert_ms": round(t_cv, 3), "i8_TMACs": round(m * n * k / t_i8 / 1e9, 1)}
        print(json.dumps(rec), flush=True)
        out.append(rec)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/gemm_i8_bench.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
