"""Pins for oracle/model.py and synth/ (CPU only)."""
import math

import numpy as np
import pytest

from oracle import model
from oracle.philox import philox4x32_10, random_action
from synth import era5_test_mask, make_workload


def test_matern_constants(golden):
    for name, nu, ell, sigma, x, expected, tol in golden("matern_constants.txt"):
        nu, ell, sigma, x, expected, tol = map(float, (nu, ell, sigma, x, expected, tol))
        if name == "A00":
            A, _, _ = model.temporal_transition(nu, ell, sigma, x)
            got = A[0, 0]
        elif name.startswith("Sinf"):
            _, _, S = model.temporal_transition(nu, ell, sigma, x)
            got = S[int(name[-2]), int(name[-1])]
        elif name == "cov_lag":
            A, _, S = model.temporal_transition(nu, ell, sigma, x)
            got = (A @ S)[0, 0]
        else:
            got = model.matern(nu, x / ell)
        assert abs(got - expected) <= tol, (name, got, expected)


@pytest.mark.parametrize("nu", [0.5, 1.5, 2.5])
def test_sde_reproduces_closed_form_kernel(nu):
    """[expm(F dt) Sigma_inf]_00 = sigma^2 Matern(nu)(dt/ell): pins F, L, q, expm, Lyapunov."""
    ell, sigma = 0.7, 2.0
    for dt in [0.0, 0.05, 0.3, 1.7]:
        A, Q, S = model.temporal_transition(nu, ell, sigma, dt)
        assert abs((A @ S)[0, 0] - sigma ** 2 * model.matern(nu, dt / ell)) < 1e-10
        assert np.min(np.linalg.eigvalsh(Q)) > -1e-10


def test_chapman_kolmogorov():
    nu, ell, sigma = 1.5, 3.0, 10.0
    A1, Q1, _ = model.temporal_transition(nu, ell, sigma, 0.4)
    A2, Q2, _ = model.temporal_transition(nu, ell, sigma, 0.6)
    A3, Q3, _ = model.temporal_transition(nu, ell, sigma, 1.0)
    assert np.allclose(A2 @ A1, A3, rtol=1e-12, atol=1e-12)
    assert np.allclose(A2 @ Q1 @ A2.T + Q2, Q3, rtol=1e-9, atol=1e-9)
    _, Q0, _ = model.temporal_transition(nu, ell, sigma, 0.0)
    assert np.allclose(Q0, 0.0, atol=1e-9)


def test_spatial_gram_psd_and_symmetry():
    rng = np.random.default_rng(0)
    X = rng.standard_normal((40, 3))
    for nu in (0.5, 1.5, 2.5):
        K = model.spatial_gram(X, X, nu, 0.8)
        assert np.allclose(K, K.T)
        assert np.allclose(np.diag(K), 1.0)
        assert np.linalg.eigvalsh(K).min() > -1e-10


def test_kronecker_lemma_b1():
    """Sigma_{k+1} = A Sigma_k A^T + Q in Kronecker form (Lemma B.1)."""
    wl = make_workload("line8")
    ssm = model.ssm_from_workload(wl)
    for k in range(1, ssm.T + 1):
        lhs = ssm.Sigma(k)
        rhs = ssm.A(k) @ ssm.Sigma(k - 1) @ ssm.A(k).T + ssm.Q(k)
        assert np.allclose(lhs, rhs, atol=1e-12)


def test_table_c1_sizes(golden):
    for f, nx, D, nk, ntot in golden("era5_table_c1.txt"):
        f = int(f)
        m = era5_test_mask(1440 // f, 720 // f + 1)
        assert m.size == int(nx) and 2 * m.size == int(D)
        assert (~m).sum() == int(nk) and 48 * (~m).sum() == int(ntot)


def test_philox_kat(golden):
    for row in golden("philox4x32_10_kat.txt"):
        vals = [int(x, 16) for x in row]
        assert philox4x32_10(vals[0:4], vals[4:6]) == tuple(vals[6:10])


def test_random_actions_moments():
    z = random_action(7, 3, 2, 200000)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01
    assert np.array_equal(z, random_action(7, 3, 2, 200000))
    assert not np.array_equal(z[:100], random_action(7, 3, 3, 100))
