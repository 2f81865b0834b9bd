"""Model layer of the oracle: temporal Matérn SDE, spatial kernels, dense LGSSM.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* Temporal prior: Matérn(nu = p + 1/2) has a finite SDE representation
  (Remark B.2).  The companion-form drift F and diffusion L q L^T are
  the standard construction the remark cites; we obtain the discrete transition
  A^t(dt) = expm(F dt) by a general matrix exponential (scipy) and the stationary
  covariance Sigma_inf by solving the continuous Lyapunov equation
  F S + S F^T + L q L^T = 0, then Q^t = Sigma_inf - A Sigma_inf A^T.  (The CUDA
  library uses closed forms instead; the two are independent.)
* Spatial prior: unit-output-scale Matérn on Euclidean distance (extrinsic on the
  sphere), Sigma = sigma^2 Matern_t (x) Matern_x.
* Lemma B.1: A = A^t (x) I, Q = Q^t (x) Sigma^x(X, X),
  Sigma_u(t_k, t_k) = Sigma^t(t_k, t_k) (x) Sigma^x(X, X); state derivative-major.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np
import scipy.linalg
from scipy.spatial.distance import cdist


# --------------------------------------------------------------------------- kernels
def matern(nu: float, r: np.ndarray) -> np.ndarray:
    """Unit-output-scale Matérn(nu) as a function of r = distance / lengthscale."""
    r = np.asarray(r, dtype=np.float64)
    if nu == 0.5:
        return np.exp(-r)
    if nu == 1.5:
        a = math.sqrt(3.0) * r
        return (1.0 + a) * np.exp(-a)
    if nu == 2.5:
        a = math.sqrt(5.0) * r
        return (1.0 + a + a * a / 3.0) * np.exp(-a)
    raise ValueError(f"unsupported Matérn nu={nu}")


def spatial_gram(X: np.ndarray, Y: np.ndarray, nu: float, ell: float) -> np.ndarray:
    """Sigma^x(X, Y) with Euclidean distance (cdist), unit output scale."""
    return matern(nu, cdist(np.atleast_2d(X), np.atleast_2d(Y)) / ell)


# --------------------------------------------------------------------------- temporal SDE
def matern_sde(nu: float, ell: float, sigma: float):
    """Companion-form SDE (F, L, q) of sigma^2 * Matérn(nu, ell), nu = p + 1/2.

    Spectral density S(w) = q / (lam^2 + w^2)^(p+1), lam = sqrt(2 nu)/ell,
    q = sigma^2 * 2 sqrt(pi) lam^(2 nu) Gamma(nu + 1/2) / Gamma(nu)
    (the rational-spectrum form of Remark B.2).
    """
    p = int(round(nu - 0.5))
    if abs(nu - (p + 0.5)) > 1e-12 or p < 0:
        raise ValueError("nu must be p + 1/2")
    lam = math.sqrt(2.0 * nu) / ell
    d = p + 1
    F = np.zeros((d, d))
    F[:-1, 1:] = np.eye(d - 1)
    # last row: -binom(d, j) lam^(d-j) for j = 0..d-1  ((d/dt + lam)^d companion form)
    for j in range(d):
        F[-1, j] = -math.comb(d, j) * lam ** (d - j)
    L = np.zeros((d, 1))
    L[-1, 0] = 1.0
    q = sigma ** 2 * 2.0 * math.sqrt(math.pi) * lam ** (2 * nu) * math.gamma(nu + 0.5) / math.gamma(nu)
    return F, L, q


def stationary_cov(F: np.ndarray, L: np.ndarray, q: float) -> np.ndarray:
    """Solve F S + S F^T + L q L^T = 0 (continuous Lyapunov)."""
    S = scipy.linalg.solve_continuous_lyapunov(F, -q * (L @ L.T))
    return 0.5 * (S + S.T)


def temporal_transition(nu: float, ell: float, sigma: float, dt: float):
    """(A^t(dt), Q^t(dt), Sigma_inf) for the stationary Matérn SDE."""
    F, L, q = matern_sde(nu, ell, sigma)
    Sinf = stationary_cov(F, L, q)
    A = scipy.linalg.expm(F * dt)
    Q = Sinf - A @ Sinf @ A.T
    return A, 0.5 * (Q + Q.T), Sinf


# --------------------------------------------------------------------------- LGSSM
@dataclasses.dataclass
class SSM:
    """Dense LGSSM in Kronecker form (Def. A.1 P:894-913 with Lemma B.1).

    Steps are k = 1..T; ``A_t[k-1]``/``Q_t[k-1]`` is the transition INTO step k.
    ``obs[k-1] = (idx, y, noise_var)`` with idx spatial indices of f_0 (H_k picks
    rows idx of block 0); an empty idx means IsMissing.
    """

    K: np.ndarray                 # Sigma^x(X, X), N_X x N_X
    sig_t0: np.ndarray            # Sigma^t(t_0, t_0), D' x D'
    mu0: np.ndarray               # D
    A_t: list
    Q_t: list
    obs: list

    @property
    def d_time(self) -> int:
        return self.sig_t0.shape[0]

    @property
    def n_space(self) -> int:
        return self.K.shape[0]

    @property
    def D(self) -> int:
        return self.d_time * self.n_space

    @property
    def T(self) -> int:
        return len(self.A_t)

    def sigma_t(self, k: int) -> np.ndarray:
        """Sigma^t_k by the recursion Sigma^t_{k} = A^t Sigma^t_{k-1} A^tT + Q^t."""
        S = self.sig_t0
        for j in range(k):
            S = self.A_t[j] @ S @ self.A_t[j].T + self.Q_t[j]
        return S

    def Sigma(self, k: int) -> np.ndarray:
        return np.kron(self.sigma_t(k), self.K)

    def A(self, k: int) -> np.ndarray:
        """Transition matrix INTO step k (A_{k-1} in the paper's indexing)."""
        return np.kron(self.A_t[k - 1], np.eye(self.n_space))

    def Q(self, k: int) -> np.ndarray:
        return np.kron(self.Q_t[k - 1], self.K)

    def H(self, k: int) -> np.ndarray:
        idx = self.obs[k - 1][0]
        H = np.zeros((len(idx), self.D))
        H[np.arange(len(idx)), idx] = 1.0
        return H

    def Lam(self, k: int) -> np.ndarray:
        return np.diag(self.obs[k - 1][2])

    def y(self, k: int) -> np.ndarray:
        return self.obs[k - 1][1]

    def missing(self, k: int) -> bool:
        return len(self.obs[k - 1][0]) == 0


def ssm_from_workload(wl, dtype_round: Optional[type] = None) -> SSM:
    """Assemble the dense LGSSM of a synth.Workload.

    ``dtype_round=np.float32`` rounds the floating inputs (coords, y, noise) to
    fp32 first so the fp64 oracle sees exactly what an fp32 device run sees (R20).
    """
    X = wl.coords
    ys = wl.y
    nvs = wl.noise_var
    if dtype_round is not None:
        X = X.astype(dtype_round).astype(np.float64)
        ys = [y.astype(dtype_round).astype(np.float64) for y in ys]
        nvs = [v.astype(dtype_round).astype(np.float64) for v in nvs]
    K = spatial_gram(X, X, wl.nu_x, wl.ell_x)
    A_t, Q_t = [], []
    Sinf = None
    for dt in wl.dts:
        A, Q, Sinf = temporal_transition(wl.nu_t, wl.ell_t, wl.sigma, float(dt))
        A_t.append(A)
        Q_t.append(Q)
    if Sinf is None:
        _, _, Sinf = temporal_transition(wl.nu_t, wl.ell_t, wl.sigma, 0.0)
    mu0 = np.zeros(Sinf.shape[0] * X.shape[0])
    obs = [(np.asarray(i, dtype=np.int64), np.asarray(y, dtype=np.float64), np.asarray(v, dtype=np.float64))
           for i, y, v in zip(wl.obs_idx, ys, nvs)]
    return SSM(K=K, sig_t0=Sinf, mu0=mu0, A_t=A_t, Q_t=Q_t, obs=obs)
