"""GPU parity of cakf_interpolate (temporal interpolation, Cor. A.10 P:1386-1437; algs
P:1445-1499) against oracle/interp.py, through the C-ABI.  The device takes its transitions
A(t, t_k), Q(t, t_k), A(t_{k+1}, t) from the library's closed forms, the oracle from expm +
Lyapunov (independent)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import cakf as ocakf  # noqa: E402
from oracle import interp, model  # noqa: E402
from paper_2405_08971_b200 import CAKF_FILTER, CAKF_SMOOTH, binding, runner  # noqa: E402
from synth import make_workload  # noqa: E402

EPS32 = float(np.finfo(np.float32).eps)


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _run(wl, dtype, keep=True):
    trans, _ = runner.transitions(wl)
    h = runner.make_handle(wl, dtype, keep_carriers=keep)
    runner.run(h, trans, runner.stage_inputs(wl, dtype), smooth=True)
    h.sync()
    return h


def _mats(wl, k, frac):
    dt = float(wl.dts[k] if k < wl.T else wl.dts[-1])
    A1, Q1, _ = binding.matern_transition(wl.nu_t, wl.ell_t, wl.sigma, frac * dt)
    A2 = binding.matern_transition(wl.nu_t, wl.ell_t, wl.sigma, (1 - frac) * dt)[0]
    oA1, oQ1, _ = model.temporal_transition(wl.nu_t, wl.ell_t, wl.sigma, frac * dt)
    oA2 = model.temporal_transition(wl.nu_t, wl.ell_t, wl.sigma, (1 - frac) * dt)[0]
    return (A1, Q1, A2), (oA1, oQ1, oA2)


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def _vrel(a, b):
    return float(np.max(np.abs(a - b) / np.abs(b)))


CASES = [("cfg1", dict(T=8, policy="cg", max_iter=5, max_rank=7)),
         ("sphere48", dict(T=5, policy="random", max_iter=8, max_rank=12)),
         ("sphere48", dict(T=5, policy="cg", max_iter=8, max_rank=-1))]


@pytest.mark.parametrize("name,kw", CASES)
def test_interpolation_fp64(name, kw):
    wl = make_workload(name, **kw)
    h = _run(wl, "f64")
    ssm, tr, sm = ocakf.run_workload(wl)
    for k, frac in [(1, 0.5), (2, 0.25), (wl.T - 1, 0.9), (wl.T, 0.4)]:
        dev, ora = _mats(wl, k, frac)
        om, ov, oms, ovs = interp.interpolate(ssm, tr, sm, k, *ora)
        fm, fv = h.interpolate(k, dev[0], dev[1], dev[2], CAKF_FILTER)
        smn, svr = h.interpolate(k, dev[0], dev[1], dev[2], CAKF_SMOOTH)
        assert _rel(fm, om) < 1e-9 and _vrel(fv, ov) < 1e-9, (k, _rel(fm, om), _vrel(fv, ov))
        assert _rel(smn, oms) < 1e-9 and _vrel(svr, ovs) < 1e-9, (k, _rel(smn, oms), _vrel(svr, ovs))
    h.destroy()


def test_interpolation_at_grid_point_is_the_stored_state():
    """A1 = I, Q1 = 0 at an untruncated step returns the step's own filter / smoother state."""
    wl = make_workload("sphere48", T=4, policy="cg", max_iter=8, max_rank=-1)
    h = _run(wl, "f64")
    I = np.eye(wl.d_time)
    for k in range(1, wl.T):
        A2 = binding.matern_transition(wl.nu_t, wl.ell_t, wl.sigma, float(wl.dts[k]))[0]
        fm, fv = h.interpolate(k, I, np.zeros_like(I), A2, CAKF_FILTER)
        gm, gv = h.get(k, CAKF_FILTER)
        assert _rel(fm, gm) < 1e-12 and _vrel(fv, gv) < 1e-12
        sm_, sv_ = h.interpolate(k, I, np.zeros_like(I), A2, CAKF_SMOOTH)
        gm, gv = h.get(k, CAKF_SMOOTH)
        assert _rel(sm_, gm) < 1e-11 and _vrel(sv_, gv) < 1e-11
    h.destroy()


def test_interpolation_fp32_cancellation_bound():
    wl = make_workload("sphere48", T=4, policy="random", max_iter=16, max_rank=24)
    h = _run(wl, "f32")
    ssm, tr, sm = ocakf.run_workload(wl, dtype_round=np.float32)
    for k, frac in [(1, 0.3), (3, 0.6)]:
        dev, ora = _mats(wl, k, frac)
        om, ov, oms, ovs = interp.interpolate(ssm, tr, sm, k, *ora)
        sdd = np.concatenate([np.full(wl.n_space, (ora[0] @ ssm.sigma_t(k) @ ora[0].T + ora[1])[d, d])
                              for d in range(wl.d_time)])
        for which, (rm, rv) in ((CAKF_FILTER, (om, ov)), (CAKF_SMOOTH, (oms, ovs))):
            gm, gv = h.interpolate(k, dev[0], dev[1], dev[2], which)
            assert _rel(gm.astype(np.float64), rm) < 1e-4
            assert np.all(np.abs(gv - rv) <= 1e-4 * rv + 2048 * EPS32 * sdd)
    h.destroy()


def test_interpolation_state_machine():
    wl = make_workload("cfg1", T=3, policy="cg", max_iter=4, max_rank=6)
    h = _run(wl, "f64", keep=False)
    dev, _ = _mats(wl, 1, 0.5)
    h.interpolate(1, dev[0], dev[1], dev[2], CAKF_FILTER)                   # filter needs no carriers
    with pytest.raises(binding.CakfError):
        h.interpolate(1, dev[0], dev[1], dev[2], CAKF_SMOOTH)              # carriers not kept
    with pytest.raises(binding.CakfError):
        h.interpolate(0, dev[0], dev[1], dev[2], CAKF_FILTER)              # k outside [1, T]
    with pytest.raises(binding.CakfError):
        h.interpolate(wl.T + 1, dev[0], dev[1], dev[2], CAKF_FILTER)
    h.destroy()
