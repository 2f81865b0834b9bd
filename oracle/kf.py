"""Exact (dense) Kalman filtering and smoothing — the definitions CAKF/CAKS reduce to.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* kalman_filter        — Thm A.2
* rts_smoother         — Thm A.4
* downdate_kf          — Prop A.3
* inverse_free_rts     — Prop A.5
* joint_conditioning   — brute-force conditioning of the stacked trajectory
                         (Lemma B.1 joint covariances P:1741, and the
                         conditional-Gaussian formula of Lemma A.7 / P:1681-1715)

States are k = 0..T: state 0 is the prior (mu0, Sigma_0); step k = 1..T predicts
with the transition into k and updates with y_k.
"""
from __future__ import annotations

import numpy as np

from .model import SSM


def _sym(P):
    return 0.5 * (P + P.T)


def kalman_filter(ssm: SSM):
    """Thm A.2: returns dict of lists m_pred, P_pred, m, P over k = 0..T.

    G_k = H P^- H^T + Lambda, K_k = P^- H^T G^-1, m = m^- + K r, P = P^- - K G K^T.
    """
    m, P = ssm.mu0.copy(), ssm.Sigma(0)
    out = {"m_pred": [m.copy()], "P_pred": [P.copy()], "m": [m.copy()], "P": [P.copy()]}
    for k in range(1, ssm.T + 1):
        A, Q = ssm.A(k), ssm.Q(k)
        m_pred = A @ m
        P_pred = _sym(A @ P @ A.T + Q)
        if ssm.missing(k):
            m, P = m_pred, P_pred
        else:
            H, Lam, y = ssm.H(k), ssm.Lam(k), ssm.y(k)
            r = y - H @ m_pred
            G = _sym(H @ P_pred @ H.T + Lam)
            Kg = np.linalg.solve(G, H @ P_pred).T          # P^- H^T G^-1
            m = m_pred + Kg @ r
            P = _sym(P_pred - Kg @ G @ Kg.T)
        out["m_pred"].append(m_pred)
        out["P_pred"].append(P_pred)
        out["m"].append(m)
        out["P"].append(P)
    return out


def rts_smoother(ssm: SSM, kf):
    """Thm A.4: G^s_k = P_k A_k^T (P^-_{k+1})^-1; backward from m^s_T = m_T."""
    T = ssm.T
    ms = [None] * (T + 1)
    Ps = [None] * (T + 1)
    ms[T], Ps[T] = kf["m"][T], kf["P"][T]
    for k in range(T - 1, -1, -1):
        A = ssm.A(k + 1)
        Gs = np.linalg.solve(kf["P_pred"][k + 1], A @ kf["P"][k]).T
        ms[k] = kf["m"][k] + Gs @ (ms[k + 1] - kf["m_pred"][k + 1])
        Ps[k] = _sym(kf["P"][k] + Gs @ (Ps[k + 1] - kf["P_pred"][k + 1]) @ Gs.T)
    return {"m": ms, "P": Ps}


def _lsqrt_inv(G):
    """V with V V^T = G^-1 (eigh-based)."""
    lam, U = np.linalg.eigh(_sym(G))
    return U / np.sqrt(lam)


def downdate_kf(ssm: SSM):
    """Prop A.3: P^-_k = Sigma_k - M^-_k M^-_k^T, P_k = Sigma_k - M_k M_k^T.

    M^-_k = A M_{k-1}, M_k = (M^-_k, P^-_k W_k), W_k = H^T V_k, V V^T = G^-1.
    Also returns w_k = H^T G^-1 r_k and W_k (the smoother carriers of Prop A.5).
    """
    D = ssm.D
    m = ssm.mu0.copy()
    M = np.zeros((D, 0))
    out = {"m_pred": [m.copy()], "m": [m.copy()], "M_pred": [M], "M": [M],
           "w": [np.zeros(D)], "W": [np.zeros((D, 0))]}
    for k in range(1, ssm.T + 1):
        A = ssm.A(k)
        Sig = ssm.Sigma(k)
        m_pred = A @ m
        M_pred = A @ M
        P_pred = Sig - M_pred @ M_pred.T
        if ssm.missing(k):
            m, M, w, W = m_pred, M_pred, np.zeros(D), np.zeros((D, 0))
        else:
            H, Lam, y = ssm.H(k), ssm.Lam(k), ssm.y(k)
            G = H @ P_pred @ H.T + Lam
            V = _lsqrt_inv(G)
            W = H.T @ V
            w = H.T @ np.linalg.solve(G, y - H @ m_pred)
            m = m_pred + P_pred @ w
            M = np.hstack([M_pred, P_pred @ W])
        out["m_pred"].append(m_pred)
        out["m"].append(m)
        out["M_pred"].append(M_pred)
        out["M"].append(M)
        out["w"].append(w)
        out["W"].append(W)
    return out


def inverse_free_rts(ssm: SSM, ddkf):
    """Prop A.5: m^s_k = m_k + P_k A_k^T w^s_{k+1},
    P^s_k = P_k - (P_k A_k^T W^s_{k+1})(...)^T with
    w^s_k = w_k + (I - W_k W_k^T P^-_k) A_k^T w^s_{k+1} and
    W^s_k = (W_k, (I - W_k W_k^T P^-_k) A_k^T W^s_{k+1}) (factor form of eq. smooth_W).
    Needs no inverse of P^- (valid with singular Sigma^x, R14).
    """
    T = ssm.T
    ms = [None] * (T + 1)
    Ps = [None] * (T + 1)
    Sig = ssm.Sigma(T)
    P_T = Sig - ddkf["M"][T] @ ddkf["M"][T].T
    ms[T], Ps[T] = ddkf["m"][T], P_T
    ws, Ws = ddkf["w"][T], ddkf["W"][T]
    for k in range(T - 1, -1, -1):
        A = ssm.A(k + 1)
        Sig = ssm.Sigma(k)
        P = Sig - ddkf["M"][k] @ ddkf["M"][k].T
        P_pred = Sig - ddkf["M_pred"][k] @ ddkf["M_pred"][k].T
        PAt = P @ A.T
        ms[k] = ddkf["m"][k] + PAt @ ws
        B = PAt @ Ws
        Ps[k] = _sym(P - B @ B.T)
        W = ddkf["W"][k]
        proj = np.eye(ssm.D) - W @ W.T @ P_pred
        ws = ddkf["w"][k] + proj @ (A.T @ ws)
        Ws = np.hstack([W, proj @ (A.T @ Ws)])
    return {"m": ms, "P": Ps}


def joint_prior(ssm: SSM):
    """Mean and covariance of the stacked trajectory (u_0, ..., u_T).

    Cov(u_i, u_j) = Sigma_u(t_i, t_i) prod_{l=i}^{j-1} A_l^T for i <= j.
    """
    T, D = ssm.T, ssm.D
    mus = [ssm.mu0]
    for k in range(1, T + 1):
        mus.append(ssm.A(k) @ mus[-1])
    C = np.zeros(((T + 1) * D, (T + 1) * D))
    for i in range(T + 1):
        Si = ssm.Sigma(i)
        blk = Si
        C[i * D:(i + 1) * D, i * D:(i + 1) * D] = Si
        for j in range(i + 1, T + 1):
            blk = blk @ ssm.A(j).T
            C[i * D:(i + 1) * D, j * D:(j + 1) * D] = blk
            C[j * D:(j + 1) * D, i * D:(i + 1) * D] = blk.T
    return np.concatenate(mus), C


def joint_conditioning(ssm: SSM, upto: int | None = None):
    """Brute force: condition the stacked trajectory on y_1..y_upto at once.

    x2 | x1 ~ N(mu2 + C21 C11^-1 (x1 - mu1), C22 - C21 C11^-1 C12).
    Returns (means (T+1) x D, marginal covariances list).
    """
    T, D = ssm.T, ssm.D
    upto = T if upto is None else upto
    mu, C = joint_prior(ssm)
    rows, ys, noise = [], [], []
    for k in range(1, upto + 1):
        if ssm.missing(k):
            continue
        idx, y, nv = ssm.obs[k - 1]
        rows.append(k * D + idx)
        ys.append(y)
        noise.append(nv)
    if not rows:
        return mu.reshape(T + 1, D), [C[k * D:(k + 1) * D, k * D:(k + 1) * D] for k in range(T + 1)]
    rows = np.concatenate(rows)
    yv = np.concatenate(ys)
    C11 = C[np.ix_(rows, rows)] + np.diag(np.concatenate(noise))
    C21 = C[:, rows]
    gain = np.linalg.solve(C11, C21.T).T
    mpost = mu + gain @ (yv - mu[rows])
    Cpost = C - gain @ C21.T
    means = mpost.reshape(T + 1, D)
    covs = [_sym(Cpost[k * D:(k + 1) * D, k * D:(k + 1) * D]) for k in range(T + 1)]
    return means, covs
