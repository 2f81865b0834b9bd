"""The matrix-free oracle (O8) reproduces the dense oracle (O4/O5): same algorithm,
different representation, so agreement must be at rounding level."""
import numpy as np
import pytest

from oracle import cakf, mfree
from synth import make_workload


@pytest.mark.parametrize("name,kw", [("line8", dict(policy="cg", max_iter=3, max_rank=4)),
                                     ("sphere48", dict(T=3, max_iter=6, max_rank=8)),
                                     ("sphere48", dict(T=2, policy="random", max_iter=5, max_rank=-1))])
@pytest.mark.parametrize("cache", [False, True])
def test_mfree_equals_dense(name, kw, cache):
    wl = make_workload(name, **kw)
    ssm, tr, sm = cakf.run_workload(wl)
    out = mfree.run_mf(wl, chunk=97, cache=cache)
    for k in range(wl.T + 1):
        for got, ref in ((out["fm"][k], tr[k].m), (out["sm"][k], sm["m"][k])):
            assert np.max(np.abs(got - ref)) <= 1e-9 * max(np.max(np.abs(ref)), 1.0)
        for got, ref in ((out["fv"][k], tr[k].var), (out["sv"][k], sm["var"][k])):
            assert np.max(np.abs(got - ref) / ref) < 1e-9


def test_gram_apply_rows_slice():
    rng = np.random.default_rng(0)
    X = rng.standard_normal((300, 3))
    b = rng.standard_normal(300)
    full = mfree.gram_apply(X, X, b, 1.5, 0.7, chunk=64)
    part = mfree.gram_apply(X, X, b, 1.5, 0.7, chunk=64, rows=(100, 230))
    assert np.allclose(full[100:230], part, rtol=1e-14, atol=1e-12)
