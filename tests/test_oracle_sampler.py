"""Pins for oracle/sampler.py (alg:cakf-caks-sampler P:1336-1358, Matheron's rule P:1150-1216,
Prop A.9):

  * zero noise (x0 = mu_0, q = 0, eps = 0): the sampler returns the CAKF / CAKS means (the
    Matheron map evaluated at the prior mean is the posterior mean);
  * the sampler is affine in its draws, so the covariance of its output is L Sigma~ L^T with L
    evaluated column by column on Sigma~^{1/2}: without truncation it equals the CAKF covariance
    Sigma_k - M_k M_k^T (filter) and the CAKS covariance Sigma_k - M^s_k M^s_k^T (smoother) for
    any policy; with full-rank unit actions these are the exact KF / RTS covariances.
"""
import numpy as np
import pytest

from oracle import cakf, kf, model, sampler
from synth import make_workload


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("policy,rank", [("cg", 7), ("random", -1), ("cg", -1)])
def test_zero_noise_sample_is_the_posterior_mean(policy, rank):
    wl = make_workload("cfg1", T=6, policy=policy, max_iter=5, max_rank=rank)
    ssm, tr, sm = cakf.run_workload(wl)
    D, T = ssm.D, ssm.T
    zq = [np.zeros((D, 1))] * T
    ze = [np.zeros((len(ssm.obs[k][0]), 1)) for k in range(T)]
    xf, xs = sampler.sample(ssm, tr, ssm.mu0[:, None], zq, ze)
    for k in range(T + 1):
        assert _rel(xf[k][:, 0], tr[k].m) < 1e-9
        assert _rel(xs[k][:, 0], sm["m"][k]) < 1e-9


def _sample_cov(ssm, tr, k_list):
    """Exact output covariance of the (affine) sampler: push Sigma~^{1/2} through it."""
    rng = np.random.default_rng(0)
    D, T = ssm.D, ssm.T
    def sqrt_psd(C):
        lam, U = np.linalg.eigh(0.5 * (C + C.T))
        return U * np.sqrt(np.clip(lam, 0.0, None))
    blocks = [("x0", sqrt_psd(ssm.Sigma(0)))]
    for k in range(1, T + 1):
        blocks.append((f"q{k}", sqrt_psd(np.kron(ssm.Q_t[k - 1], ssm.K))))
    for k in range(1, T + 1):
        blocks.append((f"e{k}", np.diag(np.sqrt(ssm.obs[k - 1][2]))))
    covf = {k: np.zeros((D, D)) for k in k_list}
    covs = {k: np.zeros((D, D)) for k in k_list}
    for name, L in blocks:
        S = L.shape[1]
        x0 = np.zeros((D, S))
        q = [np.zeros((D, S)) for _ in range(T)]
        e = [np.zeros((len(ssm.obs[k][0]), S)) for k in range(T)]
        if name == "x0":
            x0 = L
        elif name[0] == "q":
            q[int(name[1:]) - 1] = L
        else:
            e[int(name[1:]) - 1] = L
        # centred map: subtract the zero-draw output (the affine offset)
        ssm0 = model.SSM(ssm.K, ssm.sig_t0, np.zeros(D), ssm.A_t, ssm.Q_t,
                         [(o[0], np.zeros(len(o[1])), o[2]) for o in ssm.obs])
        xf, xs = sampler.sample(ssm0, tr, x0, q, e)
        for k in k_list:
            covf[k] += xf[k] @ xf[k].T
            covs[k] += xs[k] @ xs[k].T
    return covf, covs


@pytest.mark.parametrize("policy", ["cg", "random"])
def test_sample_covariance_is_the_computation_aware_posterior(policy):
    wl = make_workload("cfg1", T=4, policy=policy, max_iter=6, max_rank=-1)
    ssm, tr, sm = cakf.run_workload(wl)
    ks = [0, 1, 2, 4]
    covf, covs = _sample_cov(ssm, tr, ks)
    for k in ks:
        Pf = ssm.Sigma(k) - tr[k].M @ tr[k].M.T
        Ps = ssm.Sigma(k) - sm["M"][k] @ sm["M"][k].T
        assert _rel(covf[k], Pf) < 1e-9, (k, _rel(covf[k], Pf))
        assert _rel(covs[k], Ps) < 1e-9, (k, _rel(covs[k], Ps))


def test_full_actions_sampler_covariance_is_exact_rts():
    wl = make_workload("cfg1", T=3)
    ssm = model.ssm_from_workload(wl)
    tr = cakf.cakf_filter(ssm, "coord", wl.max_iter, -1, coord_order=wl.coord_order)
    K = kf.kalman_filter(ssm)
    R = kf.rts_smoother(ssm, K)
    covf, covs = _sample_cov(ssm, tr, [1, 2, 3])
    for k in (1, 2, 3):
        assert _rel(covf[k], K["P"][k]) < 1e-8
        assert _rel(covs[k], R["P"][k]) < 1e-8


def test_prior_draws_shapes_and_moments():
    wl = make_workload("cfg1", T=2)
    ssm = model.ssm_from_workload(wl)
    x0, q, e = sampler.prior_draws(ssm, 4000, np.random.default_rng(1))
    C = np.cov(x0)
    assert np.max(np.abs(C - ssm.Sigma(0))) < 0.1 * np.max(np.abs(ssm.Sigma(0)))
    assert len(q) == 2 and q[0].shape == (ssm.D, 4000) and e[1].shape == (len(ssm.obs[1][0]), 4000)
