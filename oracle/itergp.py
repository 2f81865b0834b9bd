"""Batch spatio-temporal GP posteriors (no state-space model involved).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* spacetime_kernel   — Sigma((t,x),(t',x')) = sigma^2 Matern_t(|t-t'|) Matern_x(|x-x'|)
                       (space-time separable prior)
* itergp_posterior   — Def. B.3: C = S (S^T (K + Lambda) S)^dagger S^T,
                       mean = K(z, Z) C y, var = K(z, z) - K(z, Z) C K(Z, z)
                       (garbled "S^T(...)S^T" read as "S^T(...)S", R21).
                       S = I gives the exact GP posterior.
* blockdiag_actions  — S = blkdiag(S_1, ..., S_T) of Prop. B.6.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg

from .model import matern


def spacetime_kernel(T1, X1, T2, X2, sigma, nu_t, ell_t, nu_x, ell_x):
    dt = np.abs(np.asarray(T1)[:, None] - np.asarray(T2)[None, :])
    dx = np.sqrt(np.maximum(((np.asarray(X1)[:, None, :] - np.asarray(X2)[None, :, :]) ** 2).sum(-1), 0.0))
    return sigma ** 2 * matern(nu_t, dt / ell_t) * matern(nu_x, dx / ell_x)


def training_set(wl, ys=None, nvs=None):
    """Stack (t_k, x) for every observation of every step (Prop B.6's Z^train)."""
    ts, xs, yv, nv = [], [], [], []
    ys = wl.y if ys is None else ys
    nvs = wl.noise_var if nvs is None else nvs
    for k in range(wl.T):
        idx = wl.obs_idx[k]
        ts.append(np.full(len(idx), wl.times[k]))
        xs.append(wl.coords[idx])
        yv.append(ys[k])
        nv.append(nvs[k])
    return np.concatenate(ts), np.concatenate(xs), np.concatenate(yv), np.concatenate(nv)


def blockdiag_actions(actions):
    """S = blkdiag(S_1, ..., S_T), S_k = N_k x n_k accepted actions (eq. B.2)."""
    return scipy.linalg.block_diag(*actions)


def itergp_posterior(wl, Ttest, Xtest, S=None, ys=None, nvs=None):
    """Mean and marginal variance at (Ttest, Xtest) of f | S^T y (zero prior mean)."""
    Tz, Xz, y, nv = training_set(wl, ys, nvs)
    kargs = (wl.sigma, wl.nu_t, wl.ell_t, wl.nu_x, wl.ell_x)
    Kzz = spacetime_kernel(Tz, Xz, Tz, Xz, *kargs) + np.diag(nv)
    Kxz = spacetime_kernel(Ttest, Xtest, Tz, Xz, *kargs)
    if S is None:
        C = np.linalg.inv(Kzz)
    else:
        inner = S.T @ Kzz @ S
        C = S @ np.linalg.pinv(0.5 * (inner + inner.T)) @ S.T
    mean = Kxz @ (C @ y)
    var = wl.sigma ** 2 - np.sum((Kxz @ C) * Kxz, axis=1)
    return mean, var
