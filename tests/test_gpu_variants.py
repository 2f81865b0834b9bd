"""Kernel variants that change only the schedule must agree bit for bit with the kernels they replace, on a
cfg3-sized run (D = 231,360; truncation at every step; K = 16 smoother products):
  * CAKF_TC_PERSIST: the truncation's M~ = F Q_r (Sec. 3.2) on the persistent, double-buffered
    3xBF16 kernel vs one tile per CTA (same K-block order, same two TMEM accumulators per tile; 1808 row
    tiles, so every CTA cycles both accumulator buffers several times);
  * CAKF_STRIP2: the alg:mfks K = N^ products (B_k t, V t, (K(X,T)V) t) on the cp.async strip
    kernel vs the register-prefetch strip kernel (same DMMA sequence per output).
  * CAKF_SMOOTH_OVERLAP: the smoother's kernel-applied carriers (K(X,T)V t and the carrier assembly) on the
    side stream beside the truncation's Gram and eigensolver vs in line (same kernels, same operands).
  * CAKF_SPLIT_RC8: the truncation's factor split into bf16 planes with 16-byte stores vs 2-byte stores;
  * CAKF_STAGE_AB: the inner loop's stages A and B (alg:update_pls lines 9-11) as one kernel vs
    two (same per-row arithmetic, same block and grid reduction order);
  * CAKF_TRUNC_OVERLAP: the filter truncation's eigensolver and M Q_r (and the next M^- = A M~) on their own
    stream beside the next update's prologue and first K1, joined before H M^- is gathered;
  * CAKF_K1_BOX: K1's exact-zero sub-tile test with the bounding-box bound added to the sphere bound (both
    are lower bounds on every pair distance, so the extra sub-tiles it skips hold exact zeros only).
The switches are read once per process, so each variant runs in its own interpreter."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from paper_2405_08971_b200 import CAKF_FILTER, CAKF_SMOOTH, runner
from synth import make_workload
wl = make_workload("cfg3", T=3, max_iter=16, max_rank=24)
trans, _ = runner.transitions(wl)
h = runner.make_handle(wl, "f32")
runner.run(h, trans, runner.stage_inputs(wl, "f32"), smooth=True)
h.sync()
out = []
for which in (CAKF_FILTER, CAKF_SMOOTH):
    for k in range(wl.T + 1):
        m, v = h.get(k, which)
        out += [m, v]
np.save(sys.argv[1], np.stack(out))
""" % ROOT


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("switch", ["CAKF_TC_PERSIST", "CAKF_STRIP2", "CAKF_SMOOTH_OVERLAP", "CAKF_SPLIT_RC8",
                                    "CAKF_STAGE_AB", "CAKF_TRUNC_OVERLAP", "CAKF_K1_BOX"])
def test_variant_bit_identical(tmp_path, switch):
    res = {}
    for flag in ("0", "1"):
        path = tmp_path / f"out{flag}.npy"
        env = dict(os.environ, **{switch: flag})
        subprocess.run([sys.executable, "-c", SCRIPT, str(path)], check=True, env=env, timeout=600)
        res[flag] = np.load(path)
    assert np.all(np.isfinite(res["1"]))
    assert np.array_equal(res["0"], res["1"])
