"""Pins for oracle/kf.py: exact KF/RTS vs brute force, closed forms, the exact GP."""
import numpy as np
import pytest

from oracle import itergp, kf, model
from synth import make_workload


def _max_err(a, b):
    return max(float(np.max(np.abs(x - y))) for x, y in zip(a, b))


def test_conjugate_update(golden):
    g = {r[0]: float(r[1]) for r in golden("conjugate_update.txt")}
    ssm = model.SSM(K=np.array([[1.0]]), sig_t0=np.array([[g["prior_var"]]]), mu0=np.array([g["prior_mean"]]),
                    A_t=[np.eye(1)], Q_t=[np.zeros((1, 1))],
                    obs=[(np.array([0]), np.array([g["y"]]), np.array([g["Lambda"]]))])
    out = kf.kalman_filter(ssm)
    assert abs(out["m"][1][0] - g["post_mean"]) < 1e-15
    assert abs(out["P"][1][0, 0] - g["post_var"]) < 1e-15


@pytest.fixture(scope="module")
def line8():
    wl = make_workload("line8")
    ssm = model.ssm_from_workload(wl)
    K = kf.kalman_filter(ssm)
    R = kf.rts_smoother(ssm, K)
    return wl, ssm, K, R


def test_kf_equals_brute_force(line8):
    wl, ssm, K, R = line8
    for k in range(1, ssm.T + 1):
        jm, jc = kf.joint_conditioning(ssm, upto=k)
        assert np.allclose(K["m"][k], jm[k], atol=1e-10)
        assert np.allclose(K["P"][k], jc[k], atol=1e-10)


def test_rts_equals_brute_force(line8):
    wl, ssm, K, R = line8
    jm, jc = kf.joint_conditioning(ssm)
    assert _max_err(R["m"], jm) < 1e-10
    assert _max_err(R["P"], jc) < 1e-10


def test_downdate_and_inverse_free_forms(line8):
    """Prop A.3 and Prop A.5 reproduce Thm A.2 / A.4."""
    wl, ssm, K, R = line8
    dd = kf.downdate_kf(ssm)
    for k in range(ssm.T + 1):
        P = ssm.Sigma(k) - dd["M"][k] @ dd["M"][k].T
        assert np.allclose(P, K["P"][k], atol=1e-10)
        assert np.allclose(dd["m"][k], K["m"][k], atol=1e-10)
    ifr = kf.inverse_free_rts(ssm, dd)
    assert _max_err(ifr["m"], R["m"]) < 1e-10
    assert _max_err(ifr["P"], R["P"]) < 1e-10


def test_rts_equals_closed_form_gp(line8):
    """The SSM route equals batch GP regression with the space-time kernel (no SDE)."""
    wl, ssm, K, R = line8
    Tt = np.repeat(wl.times, wl.n_space)
    Xt = np.tile(wl.coords, (wl.T, 1))
    gm, gv = itergp.itergp_posterior(wl, Tt, Xt)
    gm = gm.reshape(wl.T, -1)
    gv = gv.reshape(wl.T, -1)
    for k in range(1, wl.T + 1):
        assert np.allclose(gm[k - 1], R["m"][k][: wl.n_space], atol=1e-10)
        assert np.allclose(gv[k - 1], np.diag(R["P"][k])[: wl.n_space], atol=1e-10)


def test_missing_steps_and_no_data():
    wl = make_workload("line8")
    for k in range(wl.T):
        wl.obs_idx[k] = np.zeros(0, dtype=np.int64)
        wl.y[k] = np.zeros(0)
        wl.noise_var[k] = np.zeros(0)
    ssm = model.ssm_from_workload(wl)
    K = kf.kalman_filter(ssm)
    for k in range(ssm.T + 1):
        assert np.allclose(K["P"][k], ssm.Sigma(k))
        assert np.allclose(K["m"][k], 0.0)
