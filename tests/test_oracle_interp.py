"""Pins for oracle/interp.py (temporal interpolation, Cor. A.10 P:1386-1437, algs).

  * t = t_k without truncation: the interpolation returns the stored filter / smoother states;
  * a data-free time point inserted between t_k and t_{k+1} (transitions A(t,t_k), A(t_{k+1},t),
    Chapman-Kolmogorov noise) and the whole CAKF/CAKS re-run on the augmented grid: its states
    at the inserted point equal the interpolation (CG actions, with truncation);
  * full-rank unit actions, no truncation (cfg1): the interpolated states are the exact GP
    posterior at t (exact KF / RTS on the augmented grid).
"""
import numpy as np
import pytest

from oracle import cakf, interp, kf, model
from synth import make_workload


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def _split(wl, frac):
    dt = wl.dts[1] if len(wl.dts) > 1 else wl.dts[0]
    A1, Q1, _ = model.temporal_transition(wl.nu_t, wl.ell_t, wl.sigma, frac * dt)
    A2, Q2, _ = model.temporal_transition(wl.nu_t, wl.ell_t, wl.sigma, (1 - frac) * dt)
    return A1, Q1, A2, Q2


def test_interpolation_at_grid_point_returns_stored_states():
    wl = make_workload("cfg1", T=6, policy="cg", max_iter=5, max_rank=-1)
    ssm, tr, sm = cakf.run_workload(wl)
    I = np.eye(wl.d_time)
    for k in range(1, wl.T + 1):
        A2 = ssm.A_t[k] if k < wl.T else None
        m, v, ms, vs = interp.interpolate(ssm, tr, sm, k, I, np.zeros_like(I), A2)
        assert _rel(m, tr[k].m) < 1e-12 and _rel(v, tr[k].var) < 1e-12
        assert _rel(ms, sm["m"][k]) < 1e-10 and _rel(vs, sm["var"][k]) < 1e-10


@pytest.mark.parametrize("k,frac", [(2, 0.3), (5, 0.75), (7, 0.5)])
def test_interpolation_equals_augmented_grid_run(k, frac):
    wl = make_workload("cfg1", T=8, policy="cg", max_iter=5, max_rank=7)
    ssm, tr, sm = cakf.run_workload(wl)
    A1, Q1, A2, Q2 = _split(wl, frac)
    assert np.allclose(A2 @ A1, ssm.A_t[k], atol=1e-13)                 # Chapman-Kolmogorov
    assert np.allclose(A2 @ Q1 @ A2.T + Q2, ssm.Q_t[k], atol=1e-13)
    m, v, ms, vs = interp.interpolate(ssm, tr, sm, k, A1, Q1, A2)
    aug = interp.augmented_ssm(ssm, k, A1, Q1, A2, Q2)
    tra = cakf.cakf_filter(aug, "cg", wl.max_iter, wl.max_rank)
    sma = cakf.caks_smoother(aug, tra, wl.max_rank)
    j = k + 1                                                             # the inserted point
    assert _rel(m, tra[j].m) < 1e-10 and _rel(v, tra[j].var) < 1e-10
    assert _rel(ms, sma["m"][j]) < 1e-9 and _rel(vs, sma["var"][j]) < 1e-9
    # and the rest of the augmented run is the original run
    assert _rel(tra[j + 1].m, tr[k + 1].m) < 1e-9


def test_interpolation_is_exact_gp_posterior_cfg1():
    wl = make_workload("cfg1", T=10)
    ssm = model.ssm_from_workload(wl)
    tr = cakf.cakf_filter(ssm, "coord", wl.max_iter, -1, coord_order=wl.coord_order)
    sm = cakf.caks_smoother(ssm, tr, -1)
    k, frac = 4, 0.4
    A1, Q1, A2, Q2 = _split(wl, frac)
    m, v, ms, vs = interp.interpolate(ssm, tr, sm, k, A1, Q1, A2)
    aug = interp.augmented_ssm(ssm, k, A1, Q1, A2, Q2)
    K = kf.kalman_filter(aug)
    R = kf.rts_smoother(aug, K)
    assert _rel(m, K["m"][k + 1]) < 1e-9 and _rel(v, np.diag(K["P"][k + 1])) < 1e-9
    assert _rel(ms, R["m"][k + 1]) < 1e-9 and _rel(vs, np.diag(R["P"][k + 1])) < 1e-9


def test_interpolation_after_last_step_is_the_predictive():
    wl = make_workload("cfg1", T=4, policy="cg", max_iter=5, max_rank=7)
    ssm, tr, sm = cakf.run_workload(wl)
    A1, Q1, _, _ = _split(wl, 0.6)
    m, v, ms, vs = interp.interpolate(ssm, tr, sm, wl.T, A1, Q1, None)
    assert np.array_equal(m, ms) and np.array_equal(v, vs)
    Sig = np.kron(A1 @ ssm.sigma_t(wl.T) @ A1.T + Q1, ssm.K)
    M = np.kron(A1, np.eye(wl.n_space)) @ tr[wl.T].Mtil
    assert _rel(v, np.diag(Sig - M @ M.T)) < 1e-13
