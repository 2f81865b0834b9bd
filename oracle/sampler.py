"""CAKF / CAKS posterior sampler (TEST INFRASTRUCTURE ONLY).

alg:cakf-caks-sampler, i.e. Matheron's rule (Lemma) applied to the
projected state-space model of the CAKF (Prop A.9 P:1290-1313 for the inverse-free
backward recursion), densely in fp64 and with the prior draws passed in:

  forward   x_0 = xi_0 ~ N(mu_0, Sigma_0);  for k = 1..T:
              x^-_k = A_{k-1} x_{k-1} + q_{k-1}                    q_{k-1} ~ N(0, Q_{k-1})
              w_k   = H_k^T V_k V_k^T (y_k - H_k x^-_k - eps_k)    eps_k ~ N(0, Lambda_k)     (R25)
              x_k   = x^-_k + P^-_k w_k                             P^-_k = Sigma_k - M^-_k M^-_k^T
  backward  w^s_T = w_T;  for k = T-1..0:
              x^s_k = x_k + P_k A_k^T w^s_{k+1}                      P_k = Sigma_k - M_k M_k^T (R7)
              w^s_k = w_k + (I - W_k W_k^T P^-_k) A_k^T w^s_{k+1}    W_k = H_k^T V_k
            x^s_T = x_T.

R25: the paper writes the projected residual V-check^T (y-check - H-check x^- - eps-check) with
y-check = S^T y, eps-check ~ N(0, S^T Lambda S); with V = S V-check (alg:projected_update) this is
V^T (y - H x^- - eps) for a full-space eps ~ N(0, Lambda), so no actions need to be stored.
Every argument may carry several samples as columns.
"""
from __future__ import annotations

import numpy as np


def sample(ssm, trace, x0, q, eps, smoother: bool = True):
    """x0: D x S; q[k-1]: D x S (k = 1..T); eps[k-1]: N_k x S.
    Returns (filter samples x_k, smoother samples x^s_k) as lists over k = 0..T."""
    T = ssm.T
    x = np.array(x0, dtype=np.float64, copy=True)
    if x.ndim == 1:
        x = x[:, None]
    xs_f = [x]
    w = [np.zeros_like(x)]
    for k in range(1, T + 1):
        rec = trace[k]
        xp = ssm.A(k) @ x + np.asarray(q[k - 1]).reshape(x.shape)
        if rec.upd is None:                                       # IsMissing
            x, wk = xp, np.zeros_like(xp)
        else:
            H = ssm.H(k)
            V = rec.upd.V
            res = ssm.y(k)[:, None] - H @ xp - np.asarray(eps[k - 1]).reshape(-1, x.shape[1])
            wk = H.T @ (V @ (V.T @ res))
            P_pred = ssm.Sigma(k) - rec.M_pred @ rec.M_pred.T
            x = xp + P_pred @ wk
        xs_f.append(x)
        w.append(wk)
    if not smoother:
        return xs_f, None
    xs = [None] * (T + 1)
    xs[T] = xs_f[T]
    ws = w[T]
    for k in range(T - 1, -1, -1):
        rec = trace[k]
        Sig = ssm.Sigma(k)
        z = ssm.A(k + 1).T @ ws
        xs[k] = xs_f[k] + (Sig - rec.M @ rec.M.T) @ z
        P_pred = Sig - rec.M_pred @ rec.M_pred.T
        W = rec.W
        ws = w[k] + z - W @ (W.T @ (P_pred @ z))
    return xs_f, xs


def prior_draws(ssm, n_samples: int, rng):
    """Exact prior draws for small problems (eigen square roots): x0 ~ N(mu_0, Sigma_0),
    q_{k-1} ~ N(0, Q_{k-1} (x) K), eps_k ~ N(0, Lambda_k)."""
    def sqrt_psd(C):
        lam, U = np.linalg.eigh(0.5 * (C + C.T))
        return U * np.sqrt(np.clip(lam, 0.0, None))
    D, T = ssm.D, ssm.T
    L0 = sqrt_psd(ssm.Sigma(0))
    x0 = ssm.mu0[:, None] + L0 @ rng.standard_normal((D, n_samples))
    q, eps = [], []
    for k in range(1, T + 1):
        Lq = sqrt_psd(np.kron(ssm.Q_t[k - 1], ssm.K))
        q.append(Lq @ rng.standard_normal((D, n_samples)))
        nv = ssm.obs[k - 1][2]
        eps.append(np.sqrt(nv)[:, None] * rng.standard_normal((len(nv), n_samples)))
    return x0, q, eps
