"""Temporal interpolation of CAKF / CAKS states at an off-grid time (TEST INFRASTRUCTURE ONLY).

Follows Cor. A.10 in the computation-aware form of alg:cakf-interpolation
 and alg:caks-interpolation, densely, in fp64:

  t_k <= t < t_{k+1}, A1 = A(t, t_k), Q1 = Q(t, t_k), A2 = A(t_{k+1}, t):
    filter    m(t) = (A1 (x) I) m_k,   M(t) = (A1 (x) I) M~_k  (the truncated factor),
              P(t) = Sigma(t) - M(t) M(t)^T,  Sigma(t) = (A1 Sigma^t_k A1^T + Q1) (x) K_X
    smoother  (k < T)  m^s(t) = m(t) + P(t) (A2 (x) I)^T w^s_{k+1},
                       M^s(t) = [M(t), P(t) (A2 (x) I)^T W^s_{k+1}],  P^s(t) = Sigma(t) - M^s M^s^T
              (k = T)  the filter state.
  At t = t_k (A1 = I, Q1 = 0) the algorithms return the stored step-k states instead.

Only tests/ may import this module; the product path never calls it.
"""
from __future__ import annotations

import numpy as np


def interpolate(ssm, trace, sm, k: int, A1: np.ndarray, Q1: np.ndarray, A2: np.ndarray | None):
    """States at t in [t_k, t_{k+1}) (k = T: t >= t_T).  Returns (m, var, m_s, var_s)."""
    if not 1 <= k <= ssm.T:
        raise ValueError("k must be in [1, T]")
    nx = ssm.n_space
    I = np.eye(nx)
    Sig_t = A1 @ ssm.sigma_t(k) @ A1.T + Q1                       # Sigma^t(t): predict from t_k
    Sig = np.kron(Sig_t, ssm.K)
    A1k = np.kron(A1, I)
    m = A1k @ trace[k].m                                          # alg:cakf-interpolation
    M = A1k @ trace[k].Mtil
    var = np.diag(Sig) - np.sum(M * M, axis=1)                    # P(t) = Sigma(t) - M M^T
    if k == ssm.T or sm is None:
        return m, var, m.copy(), var.copy()
    P = Sig - M @ M.T
    PA2t = P @ np.kron(A2, I).T                                   # P(t) A(t_{k+1}, t)^T
    ms = m + PA2t @ sm["ws"][k + 1]                               # alg:caks-interpolation
    Ms = np.hstack([M, PA2t @ sm["Ws"][k + 1]])
    var_s = np.diag(Sig) - np.sum(Ms * Ms, axis=1)
    return m, var, ms, var_s


def augmented_ssm(ssm, k: int, A1, Q1, A2, Q2):
    """The same LGSSM with a data-free time point inserted between steps k and k+1 (pins):
    transitions A1 (t_k -> t) and A2 (t -> t_{k+1}), whose composition must equal A_{k+1}."""
    import copy
    aug = copy.copy(ssm)
    aug.A_t = list(ssm.A_t[:k]) + [A1, A2] + list(ssm.A_t[k + 1:])
    aug.Q_t = list(ssm.Q_t[:k]) + [Q1, Q2] + list(ssm.Q_t[k + 1:])
    empty = (np.zeros(0, dtype=np.int64), np.zeros(0), np.zeros(0))
    aug.obs = list(ssm.obs[:k]) + [empty] + list(ssm.obs[k:])
    return aug
