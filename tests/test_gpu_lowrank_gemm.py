"""The fp32 path's low-rank contractions (post-loop P:1532-1541, truncation Gram / M Q_r Sec. 3.2
P:334-369, smoother alg:mfks P:388-409) run on the INT8 tensor cores with exact slice products and
fp64 sums (kernels_gemm_i8.cu).  Checked through the C-ABI `cakf_lowrank_gemm` against
the fp64 product of the same fp32 inputs (numpy), element by element, relative to sum_k |a||b|."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2405_08971_b200 import binding  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return "cuda"


def _check(A, B, ta, tb, alpha, beta, C0, dev, tol):
    At, Bt = torch.tensor(A, device=dev), torch.tensor(B, device=dev)
    C = torch.tensor(C0, device=dev) if C0 is not None else None
    got = binding.lowrank_gemm(At, Bt, transa=ta, transb=tb, alpha=alpha, beta=beta, C=C).cpu().numpy()
    opA = A.astype(np.float64).T if ta else A.astype(np.float64)
    opB = B.astype(np.float64).T if tb else B.astype(np.float64)
    ref = alpha * opA @ opB
    scale = abs(alpha) * np.abs(opA) @ np.abs(opB)
    if C0 is not None and beta != 0.0:
        ref = ref + beta * C0.astype(np.float64)
        scale = scale + abs(beta) * np.abs(C0.astype(np.float64))
    # the fp32 output rounding is 2^-24 relative to |C|
    err = np.abs(got.astype(np.float64) - ref) - 2.0 ** -24 * np.abs(ref)
    # slicing bound (kernels_gemm_i8.cu): per product < 12 * 2^-35 * 2^(e_a + e_b) with 2^e <= 2 max|.|
    # over the 8192-element K chunk, i.e. < 2^-29.4 * max_chunk|a| * max_chunk|b|
    K = opA.shape[1]
    KC = 8192
    bound = np.zeros_like(ref)
    for c0 in range(0, K, KC):
        a = np.abs(opA[:, c0:c0 + KC]).max(axis=1)
        b = np.abs(opB[c0:c0 + KC, :]).max(axis=0)
        bound += min(KC, K - c0) * np.outer(a, b)
    bound *= abs(alpha) * 2.0 ** -29
    assert np.all(err <= bound + 1e-300), float(np.max(err / np.maximum(bound, 1e-300)))
    worst = float(np.max(err / np.maximum(scale, 1e-300)))
    assert worst < tol, worst
    return worst


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (37, 5, 3), (128, 96, 64), (200, 130, 16384 + 77), (513, 70, 40000),
                                   (576, 576, 33000)])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_lowrank_gemm_matches_fp64(dev, m, n, k, ta, tb):
    """Shapes with ragged tiles on every axis (128-row / 96-column tiles, 64-deep K blocks) and
    K spanning several 8192-element exact chunks; Gaussian data spanning 2^10 in magnitude
    (beyond 2^11 below a chunk maximum the slices drop bits, hence the max-relative bound)."""
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    A = rng.standard_normal((k, m) if ta else (m, k)) * np.exp2(rng.integers(-5, 5, (k, m) if ta else (m, k)))
    B = rng.standard_normal((n, k) if tb else (k, n)) * np.exp2(rng.integers(-5, 5, (n, k) if tb else (k, n)))
    _check(A.astype(np.float32), B.astype(np.float32), ta, tb, 1.0, 0.0, None, dev, 1e-7)


def test_lowrank_gemm_beta_and_structure(dev):
    """beta accumulation (the smoother's y = Sigma x - M (M^T x) form), all-zero rows / columns
    (exponent 0 chunks), one dominant element per column, and fp32 subnormal-range values."""
    rng = np.random.default_rng(5)
    m, n, k = 300, 90, 20000
    A = rng.standard_normal((m, k)).astype(np.float32)
    A[7] = 0.0
    A[:, 100] *= 1e6
    A[11] *= 1e-30
    B = rng.standard_normal((k, n)).astype(np.float32)
    B[:, 3] = 0.0
    C0 = rng.standard_normal((m, n)).astype(np.float32)
    _check(A, B, False, False, -1.0, 1.0, C0, dev, 1e-4)   # the 1e6 spike costs ~20 of the 35 slice bits


def test_lowrank_gemm_gram_cancellation(dev):
    """A tall-skinny factor whose Gram has a large dynamic range (the truncation case): every
    entry of F^T F within the slicing bound at D-scale K."""
    rng = np.random.default_rng(9)
    D, c = 231360, 40
    F = (rng.standard_normal((D, c)) * np.logspace(0, -6, c)).astype(np.float32)
    _check(F, F, True, False, 1.0, 0.0, None, dev, 1e-8)


@pytest.mark.parametrize("switch", ["CAKF_I8_SPLIT_FUSED", "CAKF_I8_STACK", "CAKF_I8_PAIR"])
def test_variant_bit_identical(tmp_path, switch):
    """Schedule-only variants are bit-identical (the slice products are exact integers in any order):
    CAKF_I8_SPLIT_FUSED — the one-pass exponent + slice kernels (i8_split_kc_kernel; i8_split_rc_kernel for a
    rows-contiguous operand with K <= 1024) vs the two-pass path; CAKF_I8_STACK — stacked-B MMAs (5 per
    k-step, levels 48 columns apart, two TMEM buffers) vs one MMA per slice pair; CAKF_I8_PAIR — CTA pairs
    sharing the A planes by TMA multicast vs one CTA per tile.  Cases: several chunks, a
    partial last chunk, K not a multiple of 16, zero rows, a NaN chunk, both orientations, the RC fallback
    beyond K = 1024, N above and below one tile."""
    import os
    import subprocess
    import sys
    script = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
from paper_2405_08971_b200 import binding
rng = np.random.default_rng(21)
outs = []
for (m, n, k, ta, tb) in [(300, 70, 20003, True, False), (129, 65, 8191, False, True), (64, 513, 9000, True, True),
                          (1000, 65, 512, True, False), (300, 129, 1000, True, False), (200, 40, 1500, True, False)]:
    A = rng.standard_normal((k, m) if ta else (m, k)).astype(np.float32)
    B = rng.standard_normal((n, k) if tb else (k, n)).astype(np.float32)
    if ta: A[:, 3] = 0.0
    else: A[3] = 0.0
    if tb: B[1, 5] = np.nan
    else: B[5, 1] = np.nan
    C = binding.lowrank_gemm(torch.tensor(A, device="cuda"), torch.tensor(B, device="cuda"), transa=ta, transb=tb)
    outs.append(C.cpu().numpy().ravel())
np.save(sys.argv[1], np.concatenate(outs))
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for flag in ("0", "1"):
        path = tmp_path / f"o{flag}.npy"
        subprocess.run([sys.executable, "-c", script, str(path)], check=True, timeout=600,
                       env=dict(os.environ, **{switch: flag}))
        res[flag] = np.load(path)
    assert np.array_equal(res["0"], res["1"], equal_nan=True)
    assert np.isnan(res["1"]).any() and np.isfinite(res["1"]).any()
