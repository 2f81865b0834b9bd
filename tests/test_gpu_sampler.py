"""GPU parity of cakf_sample (alg:cakf-caks-sampler P:1336-1358) against oracle/sampler.py on
the same prior draws, through the C-ABI."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import cakf as ocakf  # noqa: E402
from oracle import sampler as osampler  # noqa: E402
from paper_2405_08971_b200 import CAKF_FILTER, CAKF_SMOOTH, binding, runner  # noqa: E402
from synth import make_workload  # noqa: E402


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _draws(ssm, S, seed, dtype):
    x0, q, e = osampler.prior_draws(ssm, S, np.random.default_rng(seed))
    if dtype == "f32":
        x0 = x0.astype(np.float32).astype(np.float64)
        q = [a.astype(np.float32).astype(np.float64) for a in q]
        e = [a.astype(np.float32).astype(np.float64) for a in e]
    return x0, q, e


def _run(wl, dtype):
    trans, _ = runner.transitions(wl)
    h = runner.make_handle(wl, dtype)
    runner.run(h, trans, runner.stage_inputs(wl, dtype), smooth=False)
    h.sync()
    return h


def _err(dev, ref):
    return max(float(np.max(np.abs(dev[k] - ref[k])) / max(np.max(np.abs(ref[k])), 1e-300))
               for k in range(len(ref)))


@pytest.mark.parametrize("name,kw,S", [("cfg1", dict(T=6, policy="cg", max_iter=5, max_rank=7), 3),
                                       ("sphere48", dict(T=4, policy="random", max_iter=8, max_rank=12), 2),
                                       ("sphere48", dict(T=4, policy="cg", max_iter=8, max_rank=-1), 1)])
def test_sampler_fp64(name, kw, S):
    wl = make_workload(name, **kw)
    h = _run(wl, "f64")
    ssm, tr, _ = ocakf.run_workload(wl, smoother=False)
    x0, q, e = _draws(ssm, S, 7, "f64")
    eps = [e[k] for k in range(wl.T) if len(ssm.obs[k][0])]
    rf, rs = osampler.sample(ssm, tr, x0, q, e)
    df = h.sample(x0, q, eps, CAKF_FILTER)
    ds = h.sample(x0, q, eps, CAKF_SMOOTH)
    assert _err(df, rf) < 1e-9, _err(df, rf)
    assert _err(ds, rs) < 1e-9, _err(ds, rs)
    h.destroy()


def test_sampler_zero_draws_give_the_device_means():
    """x0 = mu_0, q = 0, eps = 0: the samples are the device's own CAKF / CAKS means."""
    wl = make_workload("sphere48", T=4, policy="cg", max_iter=8, max_rank=12)
    h = _run(wl, "f64")
    h.smooth()
    D, T = wl.D, wl.T
    q = [np.zeros((D, 1))] * T
    eps = [np.zeros((len(wl.obs_idx[k]), 1)) for k in range(T) if len(wl.obs_idx[k])]
    ds = h.sample(np.zeros(D), q, eps, CAKF_SMOOTH)
    df = h.sample(np.zeros(D), q, eps, CAKF_FILTER)
    for k in range(T + 1):
        fm, _ = h.get(k, CAKF_FILTER)
        sm, _ = h.get(k, CAKF_SMOOTH)
        assert np.max(np.abs(df[k][:, 0] - fm)) <= 1e-9 * np.max(np.abs(fm))
        assert np.max(np.abs(ds[k][:, 0] - sm)) <= 1e-9 * np.max(np.abs(sm))
    h.destroy()


def test_sampler_fp32():
    wl = make_workload("sphere48", T=4, policy="random", max_iter=16, max_rank=24)
    h = _run(wl, "f32")
    ssm, tr, _ = ocakf.run_workload(wl, dtype_round=np.float32, smoother=False)
    x0, q, e = _draws(ssm, 4, 3, "f32")
    eps = [e[k] for k in range(wl.T) if len(ssm.obs[k][0])]
    rf, rs = osampler.sample(ssm, tr, x0, q, e)
    ds = h.sample(x0, q, eps, CAKF_SMOOTH)
    assert _err(ds.astype(np.float64), rs) < 1e-4, _err(ds.astype(np.float64), rs)
    h.destroy()
