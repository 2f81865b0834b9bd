"""Pins for oracle/cakf.py: closed-form special cases, Prop B.6, invariants."""
import numpy as np
import pytest

from oracle import cakf, itergp, kf, model
from synth import make_workload


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.fixture(scope="module")
def cfg1():
    wl = make_workload("cfg1")
    ssm = model.ssm_from_workload(wl)
    K = kf.kalman_filter(ssm)
    R = kf.rts_smoother(ssm, K)
    tr = cakf.cakf_filter(ssm, "coord", wl.max_iter, -1, coord_order=wl.coord_order)
    sm = cakf.caks_smoother(ssm, tr, -1)
    return wl, ssm, K, R, tr, sm


def test_cfg1_kf_equals_brute_force(cfg1):
    wl, ssm, K, R, tr, sm = cfg1
    jm, jc = kf.joint_conditioning(ssm)
    for k in range(ssm.T + 1):
        assert _rel(R["m"][k], jm[k]) < 1e-9
        assert _rel(np.diag(R["P"][k]), np.diag(jc[k])) < 1e-9


def test_cfg1_cakf_equals_kf(cfg1):
    """Full-rank unit-vector actions + no truncation => CAKF == KF (Prop A.3)."""
    wl, ssm, K, R, tr, sm = cfg1
    for k in range(ssm.T + 1):
        assert _rel(tr[k].m, K["m"][k]) < 1e-9
        assert np.max(np.abs(tr[k].var - np.diag(K["P"][k])) / np.diag(K["P"][k])) < 1e-9
        if k:
            assert tr[k].upd.iters == wl.n_obs(k) and tr[k].upd.rejected == 0
            assert tr[k].upd.coord_idx == list(range(wl.n_obs(k)))


def test_cfg1_caks_equals_rts(cfg1):
    """... and CAKS == RTS (Prop A.5)."""
    wl, ssm, K, R, tr, sm = cfg1
    for k in range(ssm.T + 1):
        assert _rel(sm["m"][k], R["m"][k]) < 1e-9
        assert np.max(np.abs(sm["var"][k] - np.diag(R["P"][k])) / np.diag(R["P"][k])) < 1e-9


@pytest.mark.parametrize("policy,n_iter", [("cg", 3), ("random", 4), ("cg", 1)])
def test_caks_equals_itergp(policy, n_iter):
    """Prop B.6: without truncation CAKS marginals == iterGP with S = blkdiag(S_k)."""
    wl = make_workload("line8", policy=policy, max_iter=n_iter)
    ssm = model.ssm_from_workload(wl)
    tr = cakf.cakf_filter(ssm, policy, n_iter, -1, action_seed=5)
    sm = cakf.caks_smoother(ssm, tr, -1)
    S = itergp.blockdiag_actions([tr[k].upd.S for k in range(1, wl.T + 1)])
    Tt = np.repeat(wl.times, wl.n_space)
    Xt = np.tile(wl.coords, (wl.T, 1))
    gm, gv = itergp.itergp_posterior(wl, Tt, Xt, S=S)
    gm, gv = gm.reshape(wl.T, -1), gv.reshape(wl.T, -1)
    for k in range(1, wl.T + 1):
        assert np.allclose(sm["m"][k][: wl.n_space], gm[k - 1], atol=1e-9)
        assert np.allclose(sm["var"][k][: wl.n_space], gv[k - 1], atol=1e-9)
    # filter at the last step == iterGP given only data up to T ("suffices to run the filter")
    assert np.allclose(tr[wl.T].m[: wl.n_space], gm[-1], atol=1e-9)


def test_caks_equals_itergp_sphere():
    wl = make_workload("sphere48", T=2, max_iter=5)
    ssm = model.ssm_from_workload(wl)
    tr = cakf.cakf_filter(ssm, "cg", 5, -1)
    sm = cakf.caks_smoother(ssm, tr, -1)
    S = itergp.blockdiag_actions([tr[k].upd.S for k in range(1, wl.T + 1)])
    Tt = np.repeat(wl.times, wl.n_space)
    Xt = np.tile(wl.coords, (wl.T, 1))
    gm, gv = itergp.itergp_posterior(wl, Tt, Xt, S=S)
    gm, gv = gm.reshape(wl.T, -1), gv.reshape(wl.T, -1)
    for k in range(1, wl.T + 1):
        assert _rel(sm["m"][k][: wl.n_space], gm[k - 1]) < 1e-8
        assert _rel(sm["var"][k][: wl.n_space], gv[k - 1]) < 1e-8


def _one_step(seed=0, D=12, N=8, rank=3):
    rng = np.random.default_rng(seed)
    B = rng.standard_normal((D, D))
    Sigma = B @ B.T / D + 0.1 * np.eye(D)
    M_pred = 0.3 * rng.standard_normal((D, rank))
    while np.linalg.eigvalsh(Sigma - M_pred @ M_pred.T).min() <= 0:
        M_pred *= 0.5
    H = np.zeros((N, D))
    H[np.arange(N), rng.choice(D, N, replace=False)] = 1.0
    lam = 0.05 + 0.1 * rng.random(N)
    y = rng.standard_normal(N)
    m_pred = rng.standard_normal(D)
    return m_pred, M_pred, Sigma, H, lam, y


def test_g_orthonormality_and_galerkin():
    """V^T G V = I and V^T r = 0 after the loop."""
    m_pred, M_pred, Sigma, H, lam, y = _one_step()
    pol = cakf.make_policy("cg")
    u = cakf.update_iterative(m_pred, M_pred, Sigma, H, lam, y, pol, 1, 5)
    G = H @ (Sigma - M_pred @ M_pred.T) @ H.T + np.diag(lam)
    assert np.allclose(u.V.T @ G @ u.V, np.eye(u.V.shape[1]), atol=1e-10)
    r = (y - H @ m_pred) - G @ u.v
    assert np.allclose(u.V.T @ r, 0.0, atol=1e-10)


def test_batch_equals_iterative():
    """alg:projected_update == alg:update_pls for the same actions."""
    for seed in range(5):
        m_pred, M_pred, Sigma, H, lam, y = _one_step(seed)
        pol = cakf.make_policy("random", seed=seed + 11)
        u = cakf.update_iterative(m_pred, M_pred, Sigma, H, lam, y, pol, 2, 4)
        m, M, w, W = cakf.update_batch(m_pred, M_pred, Sigma, H, lam, y, u.S)
        assert np.allclose(m, u.m, atol=1e-10)
        assert np.allclose(M @ M.T, u.M @ u.M.T, atol=1e-10)
        assert np.allclose(w, u.w, atol=1e-10)


def test_cg_exact_termination_equals_kalman_update():
    m_pred, M_pred, Sigma, H, lam, y = _one_step(3)
    N = len(y)
    u = cakf.update_iterative(m_pred, M_pred, Sigma, H, lam, y, cakf.make_policy("cg"), 1, N)
    assert u.res_final <= 1e-8 * u.res0
    P_pred = Sigma - M_pred @ M_pred.T
    G = H @ P_pred @ H.T + np.diag(lam)
    Kg = P_pred @ H.T @ np.linalg.inv(G)
    assert np.allclose(u.m, m_pred + Kg @ (y - H @ m_pred), atol=1e-10)
    assert np.allclose(Sigma - u.M @ u.M.T, P_pred - Kg @ G @ Kg.T, atol=1e-10)


def test_cg_residuals_and_variances_monotone():
    m_pred, M_pred, Sigma, H, lam, y = _one_step(4)
    prev = None
    for n in range(0, len(y) + 1):
        u = cakf.update_iterative(m_pred, M_pred, Sigma, H, lam, y, cakf.make_policy("cg"), 1, n)
        var = np.diag(Sigma - u.M @ u.M.T)
        if prev is not None:
            assert np.all(var <= prev + 1e-12)
        prev = var


def test_truncation_worked_example_and_eckart_young():
    M = np.array([[3.0, 0.0], [0.0, 2.0], [0.0, 0.0]])
    Mt, dropped = cakf.truncate(M, 1)
    assert abs(np.sum(Mt ** 2) - 9.0) < 1e-12 and np.allclose(dropped, [4.0])
    assert np.allclose(np.abs(Mt[:, 0]), [3, 0, 0])
    rng = np.random.default_rng(1)
    M = rng.standard_normal((8, 5))
    Mt, dropped = cakf.truncate(M, 3)
    sv = np.linalg.svd(M, compute_uv=False)
    err = np.linalg.norm(M @ M.T - Mt @ Mt.T, "fro")
    assert abs(err - np.sqrt(np.sum(sv[3:] ** 4))) < 1e-10
    assert np.allclose(np.sort(dropped), np.sort(sv[3:] ** 2))
    # conservativeness: the represented covariance's diagonal never decreases
    assert np.all(np.sum(Mt ** 2, axis=1) <= np.sum(M ** 2, axis=1) + 1e-12)
    Mt2, d2 = cakf.truncate(M, 7)
    assert Mt2 is M and d2.size == 0


def test_no_iterations_and_uninformative_data():
    m_pred, M_pred, Sigma, H, lam, y = _one_step(5)
    u = cakf.update_iterative(m_pred, M_pred, Sigma, H, lam, y, cakf.make_policy("cg"), 1, 0)
    assert np.allclose(u.m, m_pred) and u.M.shape[1] == M_pred.shape[1]
    u = cakf.update_iterative(m_pred, M_pred, Sigma, H, lam * 1e12, y, cakf.make_policy("cg"), 1, 4)
    assert np.allclose(u.m, m_pred, atol=1e-9) and np.linalg.norm(u.M[:, M_pred.shape[1]:]) < 1e-5


@pytest.mark.parametrize("rank", [-1, 3])
def test_dominance_over_exact_posterior(rank):
    """P^_k - P_k >= 0 and P^s_k - P^s_k(exact) >= 0 (computation-awareness)."""
    wl = make_workload("line8", max_iter=2, policy="cg")
    ssm = model.ssm_from_workload(wl)
    K = kf.kalman_filter(ssm)
    R = kf.rts_smoother(ssm, K)
    tr = cakf.cakf_filter(ssm, "cg", 2, rank)
    sm = cakf.caks_smoother(ssm, tr, rank)
    for k in range(ssm.T + 1):
        Pf = ssm.Sigma(k) - tr[k].M @ tr[k].M.T
        Ps = ssm.Sigma(k) - sm["M"][k] @ sm["M"][k].T
        assert np.linalg.eigvalsh(Pf - K["P"][k]).min() > -1e-10
        assert np.linalg.eigvalsh(Ps - R["P"][k]).min() > -1e-10
        assert np.allclose(sm["var"][k], np.diag(Ps))


def test_missing_steps_give_prior():
    wl = make_workload("line8", policy="cg", max_iter=3)
    for k in range(wl.T):
        wl.obs_idx[k] = np.zeros(0, dtype=np.int64)
        wl.y[k] = np.zeros(0)
        wl.noise_var[k] = np.zeros(0)
    ssm = model.ssm_from_workload(wl)
    tr = cakf.cakf_filter(ssm, "cg", 3, 2)
    sm = cakf.caks_smoother(ssm, tr, 2)
    for k in range(ssm.T + 1):
        assert np.allclose(tr[k].m, 0) and np.allclose(sm["var"][k], np.diag(ssm.Sigma(k)))


def test_blockres_policy_pins():
    """The adaptive block policy (alg:projected_update's batch Policy call per block of b actions):
    b = 1 is CG exactly; for any b each block of actions spans the block-start residual (the actions sum to it),
    and the iterative update on the recorded actions equals alg:projected_update on them."""
    from oracle import cakf
    from oracle.model import ssm_from_workload
    from synth import make_workload
    wl = make_workload("line8", policy="cg", max_iter=5, max_rank=-1, T=2)
    ssm = ssm_from_workload(wl)
    tr_cg = cakf.cakf_filter(ssm, "cg", 5)
    tr_b1 = cakf.cakf_filter(ssm, "blockres", 5, block=1)
    for a, b in zip(tr_cg, tr_b1):
        assert np.array_equal(a.m, b.m) and np.array_equal(a.var, b.var)
    wl = make_workload("sphere48", T=2, max_iter=9, max_rank=-1)
    ssm = ssm_from_workload(wl)
    tr = cakf.cakf_filter(ssm, "blockres", 9, block=3)
    for k in (1, 2):
        rec = tr[k]
        S = rec.upd.S
        assert S.shape[1] == 9 - rec.upd.rejected
        # each block's actions are disjointly supported pieces of one residual
        for blk in range(3):
            cols = S[:, 3 * blk:3 * blk + 3]
            assert np.all(np.count_nonzero(cols, axis=1) <= 1)
        m, M, w, W = cakf.update_batch(rec.m_pred, rec.M_pred, ssm.Sigma(k), ssm.H(k), ssm.obs[k - 1][2], ssm.y(k), S)
        assert np.allclose(m, rec.m, rtol=1e-9, atol=1e-9 * np.max(np.abs(rec.m)))
        P1 = ssm.Sigma(k) - M @ M.T
        P2 = ssm.Sigma(k) - rec.M @ rec.M.T
        assert np.allclose(np.diag(P1), np.diag(P2), rtol=1e-8)
