"""Matrix-free CAKF / CAKS oracle (O8) — same algorithm as oracle/cakf.py, no D x D arrays.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Only the representation changes: products with Sigma_k = Sigma^t_k (x) Sigma^x(X, X)
are formed by generating kernel rows in chunks (``gram_apply``), P^-_k x = Sigma_k x -
M^- (M^-T x) (Prop A.3), G s = H P^- H^T s + Lambda s.  Used for state
dimensions where dense matrices do not fit (cfg3: D = 231,360) — the CPU baseline
and sampled full-size parity — and cross-checked against the dense oracle.
Readings R1-R8, R19 exactly as in oracle/cakf.py.
"""
from __future__ import annotations

import numpy as np
from scipy.spatial.distance import cdist

from .model import matern, temporal_transition


def gram_apply(Xr, Xc, B, nu, ell, chunk=1024, rows=None):
    """K(Xr, Xc) @ B, kernel rows generated `chunk` at a time (never stored).

    ``rows`` restricts the output to a row range (used for bounded timing samples).
    """
    B = np.asarray(B, dtype=np.float64)
    vec = B.ndim == 1
    if vec:
        B = B[:, None]
    r0, r1 = (0, len(Xr)) if rows is None else rows
    out = np.empty((r1 - r0, B.shape[1]))
    for i0 in range(r0, r1, chunk):
        i1 = min(r1, i0 + chunk)
        K = matern(nu, cdist(Xr[i0:i1], Xc) / ell)
        out[i0 - r0:i1 - r0] = K @ B
    return out[:, 0] if vec else out


class MFModel:
    """Kronecker LGSSM accessed only through products (Lemma B.1).

    cache=True keeps the kernel matrices K(X_T, X_T), K(X, X_T) (per observation set) and
    K(X, X) once generated instead of regenerating their rows for every product: the same
    entries (``matern(cdist(.)/ell)``, as in ``gram_apply``) and the same products, only
    stored — for D ~ 1e4 parity runs (cfg2) where regenerating rows dominates the oracle's time.
    """

    def __init__(self, wl, dtype_round=None, chunk=1024, cache=False):
        X = wl.coords
        self.ys, self.nvs = wl.y, wl.noise_var
        if dtype_round is not None:
            X = X.astype(dtype_round).astype(np.float64)
            self.ys = [y.astype(dtype_round).astype(np.float64) for y in self.ys]
            self.nvs = [v.astype(dtype_round).astype(np.float64) for v in self.nvs]
        self.X = X
        self.nu, self.ell, self.chunk = wl.nu_x, wl.ell_x, chunk
        self.idx = [np.asarray(i, dtype=np.int64) for i in wl.obs_idx]
        self.NX = len(X)
        self.At, self.Qt = [], []
        Sinf = None
        for dt in wl.dts:
            A, Q, Sinf = temporal_transition(wl.nu_t, wl.ell_t, wl.sigma, float(dt))
            self.At.append(A)
            self.Qt.append(Q)
        self.St = [Sinf]
        for A, Q in zip(self.At, self.Qt):
            self.St.append(A @ self.St[-1] @ A.T + Q)
        self.Dp = Sinf.shape[0]
        self.D = self.Dp * self.NX
        self.T = len(self.At)
        self.cache = cache
        self._K = {}

    def _kmat(self, key, Xr, Xc):
        if key not in self._K:
            self._K[key] = matern(self.nu, cdist(Xr, Xc) / self.ell)
        return self._K[key]

    def _obs_key(self, k):
        return self.idx[k - 1].tobytes()

    def ktt_apply(self, k, x):
        """K(X_T, X_T) x for the observed points of step k."""
        Xt = self.X[self.idx[k - 1]]
        if self.cache:
            return self._kmat(("TT", self._obs_key(k)), Xt, Xt) @ x
        return gram_apply(Xt, Xt, x, self.nu, self.ell, self.chunk)

    def kxt_apply(self, k, Vm):
        """K(X, X_T) Vm for the observed points of step k."""
        Xt = self.X[self.idx[k - 1]]
        if self.cache:
            return self._kmat(("XT", self._obs_key(k)), self.X, Xt) @ Vm
        return gram_apply(self.X, Xt, Vm, self.nu, self.ell, self.chunk)

    def kxx_apply(self, B):
        if self.cache:
            return self._kmat("XX", self.X, self.X) @ B
        return gram_apply(self.X, self.X, B, self.nu, self.ell, self.chunk)

    def blocks(self, Xm):
        return Xm.reshape(self.Dp, self.NX, -1)

    def sigma_apply(self, k, Xm):
        """(Sigma^t_k (x) K) Xm for Xm of shape D x m."""
        Bl = self.blocks(Xm)
        KB = [self.kxx_apply(Bl[e]) for e in range(self.Dp)]
        S = self.St[k]
        out = [sum(S[d, e] * KB[e] for e in range(self.Dp)) for d in range(self.Dp)]
        return np.concatenate(out, axis=0)

    def sigma_HT_apply(self, k, Vm):
        """Sigma_k H^T Vm (Vm: N x m): only the kernel columns of observed points."""
        Kx = self.kxt_apply(k, Vm)
        S = self.St[k]
        return np.concatenate([S[d, 0] * Kx for d in range(self.Dp)], axis=0)

    def A_apply(self, k, Xm, transpose=False):
        """(A^t (x) I) Xm with A^t the transition INTO step k."""
        A = self.At[k - 1].T if transpose else self.At[k - 1]
        Bl = self.blocks(Xm)
        out = np.concatenate([sum(A[d, e] * Bl[e] for e in range(self.Dp)) for d in range(self.Dp)], axis=0)
        return out[:, 0] if Xm.ndim == 1 else out

    def diag_sigma(self, k):
        return np.concatenate([np.full(self.NX, self.St[k][d, d]) for d in range(self.Dp)])


def _truncate(M, r):
    c = M.shape[1]
    if r < 0 or c <= r:
        return M
    lam, Q = np.linalg.eigh(M.T @ M)
    return M @ Q[:, c - r:]


def update_mf(mm: MFModel, k, m_pred, M_pred, policy, max_iter, eps=np.finfo(np.float64).eps, cgs2=True):
    """alg:update_pls with matrix-free G s = sig00 K_TT s - HM (HM^T s) + Lambda s."""
    idx = mm.idx[k - 1]
    y, lam = mm.ys[k - 1], mm.nvs[k - 1]
    HM = M_pred[idx]
    s00 = mm.St[k][0, 0]

    def G(x):
        return s00 * mm.ktt_apply(k, x) - HM @ (HM.T @ x) + lam * x

    N = len(y)
    v = np.zeros(N)
    V = np.zeros((N, 0))
    r = y - m_pred[idx]
    n = min(int(max_iter), N)
    for i in range(1, n + 1):
        s = policy(k, i, r, N)
        alpha = s @ r
        Gs = G(s)
        d = s - V @ (V.T @ Gs)
        if cgs2:
            d = d - V @ (V.T @ G(d))
        Gd = G(d)
        eta = s @ Gd
        if eta <= 64.0 * eps * abs(s @ Gs):
            V = np.hstack([V, np.zeros((N, 1))])
            continue
        v = v + (alpha / eta) * d
        V = np.hstack([V, (d / np.sqrt(eta))[:, None]])
        r = r - (alpha / eta) * Gd
    XV = np.hstack([v[:, None], V])
    PX = mm.sigma_HT_apply(k, XV) - M_pred @ (HM.T @ XV)      # P^- H^T [v V]
    m = m_pred + PX[:, 0]
    M = np.hstack([M_pred, PX[:, 1:]])
    return m, M, v, V


def run_mf(wl, dtype_round=None, smoother=True, chunk=1024, cache=False, perturb_y=0.0):
    """Full CAKF (+ CAKS) through matrix-free products; returns per-step means/variances.

    perturb_y: relative perturbation y <- y (1 + perturb_y) of every observation (the oracle's own
    input sensitivity, used to judge trajectory-sensitive comparisons such as fp64 CG at cfg2)."""
    from .cakf import make_policy
    mm = MFModel(wl, dtype_round, chunk, cache=cache)
    if perturb_y:
        mm.ys = [y * (1.0 + perturb_y) for y in mm.ys]
    pol = make_policy(wl.policy, wl.coord_order, wl.action_seed,
                      max(1, min(getattr(wl, "block_actions", 1), 1 + wl.max_iter)))
    D = mm.D
    m = np.zeros(D)
    Mt = np.zeros((D, 0))
    rec = [dict(m=m, M=Mt, Mp=Mt, v=None, V=None, var=mm.diag_sigma(0))]
    for k in range(1, mm.T + 1):
        m_pred = mm.A_apply(k, m)
        M_pred = mm.A_apply(k, Mt)
        if len(mm.idx[k - 1]) == 0:
            m, M, v, V = m_pred, M_pred, None, None
        else:
            m, M, v, V = update_mf(mm, k, m_pred, M_pred, pol, wl.max_iter, cgs2=wl.reorth)
        rec.append(dict(m=m, M=M, Mp=M_pred, v=v, V=V, var=mm.diag_sigma(k) - np.sum(M * M, axis=1)))
        Mt = _truncate(M, wl.max_rank)
    out = {"fm": [r["m"] for r in rec], "fv": [r["var"] for r in rec]}
    if not smoother:
        return out
    T = mm.T
    sm, sv = [None] * (T + 1), [None] * (T + 1)
    sm[T], sv[T] = rec[T]["m"], rec[T]["var"]

    def HT(k, Vm):
        Z = np.zeros((D, Vm.shape[1]))
        Z[mm.idx[k - 1]] = Vm
        return Z

    if rec[T]["V"] is None:
        ws, Ws = np.zeros(D), np.zeros((D, 0))
    else:
        ws, Ws = HT(T, rec[T]["v"][:, None])[:, 0], HT(T, rec[T]["V"])
    for k in range(T - 1, -1, -1):
        X = mm.A_apply(k + 1, np.hstack([ws[:, None], Ws]), transpose=True)   # A_k^T [w^s, W^s]
        y = mm.sigma_apply(k, X) - rec[k]["Mp"] @ (rec[k]["Mp"].T @ X)      # P^-_k x
        if k == 0 or rec[k]["V"] is None:
            Px, t = y, None
        else:
            Vk = rec[k]["V"]
            t = Vk.T @ y[mm.idx[k - 1]]
            Px = y - rec[k]["M"][:, rec[k]["Mp"].shape[1]:] @ t              # P_k x
        sm[k] = rec[k]["m"] + Px[:, 0]
        sv[k] = rec[k]["var"] - np.sum(Px[:, 1:] ** 2, axis=1)
        proj = X.copy()
        if t is not None:
            proj -= HT(k, rec[k]["V"] @ t)                                   # (I - W W^T P^-) x
            ws = HT(k, rec[k]["v"][:, None])[:, 0] + proj[:, 0]
            Ws = np.hstack([HT(k, rec[k]["V"]), proj[:, 1:]])
        else:
            ws, Ws = proj[:, 0], proj[:, 1:]
        Ws = _truncate(Ws, wl.max_rank)
    out["sm"], out["sv"] = sm, sv
    return out
