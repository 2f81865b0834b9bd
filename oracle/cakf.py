"""Dense CAKF / CAKS — the paper's algorithms written out literally (fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* update_iterative  — alg:update_pls, readings R1, R2, R18, R19
* update_batch      — alg:projected_update, Lemma B.2 pseudo-inverse
* truncate          — Sec. 3.2, readings R3, R4
* cakf_filter       — alg:mfkf
* caks_smoother     — alg:mfks, readings R6, R7

Covariances are formed DENSELY here (P^- = Sigma - M^- M^-T as a D x D array),
which is exactly what the matrix-free device path must never do.  Readings:
  R1  the CG policy uses the residual at the current iterate r^(i) = r^(0) - G v^(i-1)
      (P:1518), evaluated by the recurrence
      r^(i+1) = r^(i) - (alpha_i/eta_i) G d_i (identical in exact arithmetic; both sides
      use it so that ill-conditioned CG runs stay comparable).
  R19 Gram-Schmidt: line 11 as printed is one classical pass; with reorth=True (default)
      a second pass d <- d - V (V^T G d) follows (CGS2).  Identical in exact arithmetic;
      the single pass loses G-orthogonality of V in fp32 on ERA5-shaped problems.
  R2  StoppingCriterion: i = min(N^max, N_k) iterations (int count); if rtol > 0
      also stop once ||r^(i)|| <= rtol ||r^(0)||.  An action with
      eta <= 64 eps |s^T G s| is rejected: v is not updated, V gets a zero column
      (so M_k always has rank_in + iters columns and ranks are integer functions of
      (r, N^max, k)), it is counted, and the iteration still counts.
  R3/R4  Truncate keeps the top min(r, cols) eigen-directions of M^T M:
      M~ = M Q_r (same subspace as the thin SVD).
  R6  the smoother truncates W^s_k with the same procedure and cap.
  R7  P_k in the smoother uses the untruncated M_k; P^-_k uses M^-_k = A M~_{k-1}.
  R8  state 0 is the prior; step k = 1..T predicts then updates.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Optional

import numpy as np

from .model import SSM
from .philox import random_action


# --------------------------------------------------------------------------- policies
def make_policy(kind: str, coord_order=None, seed: int = 1, block: int = 1):
    """Policy(k, i, r^(i), n) -> action s (App. C.3).

    cg       : s = r^(i)                    (CG/Lanczos actions)
    coord    : s = e_{order_k[i-1]}          (coordinate actions)
    random   : s ~ N(0, I) via Philox (R16) (randomized actions)
    blockres : a block of b actions chosen at once from the residual at the block's start i0 = 1, 1+b, ...
               (the batch Policy call of alg:projected_update, repeated per block):
               s_{i0+j} = r^(i0) * 1[floor(u b / n) == j] for observation u = 0..n-1; b = 1 is CG
    """
    if kind == "cg":
        return lambda k, i, r, n: r.copy()
    if kind == "blockres":
        state = {}

        def pol(k, i, r, n):
            j = (i - 1) % block
            if j == 0:
                state["r0"] = r.copy()
            region = (np.arange(n, dtype=np.int64) * block) // n
            return np.where(region == j, state["r0"], 0.0)
        return pol
    if kind == "coord":
        def pol(k, i, r, n):
            s = np.zeros(n)
            s[int(coord_order[k - 1][i - 1])] = 1.0
            return s
        return pol
    if kind == "random":
        return lambda k, i, r, n: random_action(seed, k, i, n)
    raise ValueError(kind)


# --------------------------------------------------------------------------- update
@dataclasses.dataclass
class UpdateResult:
    m: np.ndarray
    M: np.ndarray
    w: np.ndarray
    W: np.ndarray
    v: np.ndarray            # v^(N) in observation space
    V: np.ndarray            # N x n_accepted, G-orthonormal
    S: np.ndarray            # N x n_accepted accepted actions
    iters: int
    rejected: int
    res0: float
    res_final: float
    eta_min: float
    coord_idx: list          # positions chosen by a coordinate policy (accepted or not)


def update_iterative(m_pred, M_pred, Sigma, H, lam_diag, y, policy, k, max_iter,
                     rtol=0.0, eps=np.finfo(np.float64).eps, cgs2=True) -> UpdateResult:
    """alg:update_pls, dense."""
    P_pred = Sigma - M_pred @ M_pred.T                        # line 2
    G = H @ P_pred @ H.T + np.diag(lam_diag)                  # line 3
    N = len(y)
    v = np.zeros(N)                                           # line 4
    V = np.zeros((N, 0))                                      # line 5
    r0 = y - H @ m_pred                                       # line 6
    S = []
    rejected = 0
    eta_min = np.inf
    coord_idx = []
    res0 = float(np.linalg.norm(r0))
    r = r0.copy()                                             # line 9 at i = 1
    nmax = min(int(max_iter), N)
    i = 0
    while i < nmax:                                           # line 7, R2
        if rtol > 0 and np.linalg.norm(r) <= rtol * res0:
            break
        i += 1
        s = policy(k, i, r, N)                                # line 8
        if np.count_nonzero(s) == 1:
            coord_idx.append(int(np.flatnonzero(s)[0]))
        alpha = s @ r                                         # line 10
        Gs = G @ s
        d = s - V @ (V.T @ Gs)                                # line 11
        if cgs2:
            d = d - V @ (V.T @ (G @ d))
        Gd = G @ d
        eta = s @ Gd                                          # line 12
        if eta <= 64.0 * eps * abs(s @ Gs):                   # R2 rejection: zero column
            rejected += 1
            V = np.hstack([V, np.zeros((N, 1))])
            continue
        eta_min = min(eta_min, eta)
        v = v + (alpha / eta) * d                             # line 13
        V = np.hstack([V, (d / np.sqrt(eta))[:, None]])       # line 14
        r = r - (alpha / eta) * Gd                            # line 9 for i + 1 (R1)
        S.append(s)
    r_final = r
    w = H.T @ v                                               # line 16
    W = H.T @ V                                               # line 17
    m = m_pred + P_pred @ w                                   # line 18
    M = np.hstack([M_pred, P_pred @ W])                       # line 19
    Smat = np.stack(S, axis=1) if S else np.zeros((N, 0))
    return UpdateResult(m=m, M=M, w=w, W=W, v=v, V=V, S=Smat, iters=i, rejected=rejected,
                        res0=res0, res_final=float(np.linalg.norm(r_final)),
                        eta_min=float(eta_min), coord_idx=coord_idx)


def _lsqrt_pinv(G, rcond=1e-12):
    """V with V V^T = G^dagger (symmetric eigendecomposition, relative cutoff)."""
    lam, U = np.linalg.eigh(0.5 * (G + G.T))
    keep = lam > rcond * max(lam.max(initial=0.0), 0.0)
    return U[:, keep] / np.sqrt(lam[keep])


def update_batch(m_pred, M_pred, Sigma, H, lam_diag, y, S):
    """alg:projected_update for a given action matrix S (N x n)."""
    P_pred = Sigma - M_pred @ M_pred.T
    Hc = S.T @ H                                              # H-check
    Lc = S.T @ np.diag(lam_diag) @ S                          # Lambda-check
    yc = S.T @ y                                              # y-check
    Gc = Hc @ P_pred @ Hc.T + Lc                              # G-check
    Gp = np.linalg.pinv(0.5 * (Gc + Gc.T))
    Vc = _lsqrt_pinv(Gc)
    w = Hc.T @ Gp @ (yc - Hc @ m_pred)
    W = Hc.T @ Vc
    m = m_pred + P_pred @ w
    M = np.hstack([M_pred, P_pred @ W])
    return m, M, w, W


# --------------------------------------------------------------------------- truncate
def truncate(M: np.ndarray, max_rank: int):
    """Sec. 3.2: keep the top-r eigen-directions of M^T M (R3/R4).

    Returns (M~, dropped eigenvalues ascending).  M M^T = M~ M~^T + N N^T with
    N = M Q_dropped.
    """
    c = M.shape[1]
    if max_rank < 0 or c <= max_rank:
        return M, np.zeros(0)
    lam, Q = np.linalg.eigh(M.T @ M)                          # ascending
    nd = c - max_rank
    return M @ Q[:, nd:], lam[:nd]


# --------------------------------------------------------------------------- filter
@dataclasses.dataclass
class StepRecord:
    k: int
    m_pred: np.ndarray
    m: np.ndarray
    M_pred: np.ndarray
    M: np.ndarray            # untruncated M_k (R7)
    Mtil: np.ndarray         # truncated
    w: np.ndarray
    W: np.ndarray
    var_pred: np.ndarray
    var: np.ndarray
    upd: Optional[UpdateResult]
    dropped: np.ndarray


def cakf_filter(ssm: SSM, policy_kind="cg", max_iter=64, max_rank=-1, coord_order=None,
                action_seed=1, rtol=0.0, eps=np.finfo(np.float64).eps, cgs2=True, block=1):
    """alg:mfkf: predict, Update unless IsMissing, Truncate."""
    policy = make_policy(policy_kind, coord_order, action_seed, block)
    D = ssm.D
    m = ssm.mu0.copy()
    Sig0 = ssm.Sigma(0)
    Mtil = np.zeros((D, 0))                                   # line 2
    trace = [StepRecord(0, m.copy(), m.copy(), Mtil, Mtil, Mtil, np.zeros(D), np.zeros((D, 0)),
                        np.diag(Sig0).copy(), np.diag(Sig0).copy(), None, np.zeros(0))]
    for k in range(1, ssm.T + 1):
        A = ssm.A(k)
        Sig = ssm.Sigma(k)
        m_pred = A @ m                                        # line 4 (b = 0, R9)
        M_pred = A @ Mtil                                     # line 5
        if ssm.missing(k):                                    # lines 6-10
            m, M, w, W, upd = m_pred, M_pred, np.zeros(D), np.zeros((D, 0)), None
        else:
            upd = update_iterative(m_pred, M_pred, Sig, ssm.H(k), ssm.obs[k - 1][2], ssm.y(k),
                                   policy, k, max_iter, rtol=rtol, eps=eps, cgs2=cgs2)
            m, M, w, W = upd.m, upd.M, upd.w, upd.W
        Mtil, dropped = truncate(M, max_rank)                 # line 11
        var_pred = np.diag(Sig) - np.sum(M_pred * M_pred, axis=1)
        var = np.diag(Sig) - np.sum(M * M, axis=1)
        trace.append(StepRecord(k, m_pred, m, M_pred, M, Mtil, w, W, var_pred, var, upd, dropped))
    return trace


# --------------------------------------------------------------------------- smoother
def caks_smoother(ssm: SSM, trace, max_rank=-1):
    """alg:mfks.  Returns dict with means, variances, factors M^s_k."""
    T = ssm.T
    ms = [None] * (T + 1)
    var = [None] * (T + 1)
    Ms = [None] * (T + 1)
    ranks = [0] * (T + 1)
    ws = trace[T].w                                           # line 2
    Ws = trace[T].W                                           # line 3
    ws_k = [None] * (T + 1)                                   # carriers kept for interpolation
    Ws_k = [None] * (T + 1)                                   # (alg:caks-interpolation)
    ws_k[T], Ws_k[T] = ws, Ws
    ms[T] = trace[T].m
    Ms[T] = trace[T].M
    var[T] = trace[T].var
    ranks[T] = Ws.shape[1]
    for k in range(T - 1, -1, -1):                            # line 4
        A = ssm.A(k + 1)                                      # A_k: k -> k+1
        Sig = ssm.Sigma(k)
        rec = trace[k]
        P = Sig - rec.M @ rec.M.T                             # P^_k (R7)
        P_pred = Sig - rec.M_pred @ rec.M_pred.T              # P^-_k
        PAt = P @ A.T
        ms[k] = rec.m + PAt @ ws                              # line 5
        Ms[k] = np.hstack([rec.M, PAt @ Ws])                  # line 6
        var[k] = np.diag(Sig) - np.sum(Ms[k] * Ms[k], axis=1)
        proj = np.eye(ssm.D) - rec.W @ (rec.W.T @ P_pred)
        ws = rec.w + proj @ (A.T @ ws)                        # line 7
        Ws_full = np.hstack([rec.W, proj @ (A.T @ Ws)])       # line 8
        Ws, _ = truncate(Ws_full, max_rank)                   # line 9 (R6)
        ranks[k] = Ws.shape[1]
        ws_k[k], Ws_k[k] = ws, Ws
    return {"m": ms, "var": var, "M": Ms, "rank": ranks, "ws": ws_k, "Ws": Ws_k}


def run_workload(wl, dtype_round=None, max_rank=None, smoother=True):
    """Convenience: dense CAKF (+ CAKS) on a synth.Workload."""
    from .model import ssm_from_workload
    ssm = ssm_from_workload(wl, dtype_round=dtype_round)
    mr = wl.max_rank if max_rank is None else max_rank
    tr = cakf_filter(ssm, wl.policy, wl.max_iter, mr, coord_order=wl.coord_order,
                     action_seed=wl.action_seed, rtol=wl.rtol, cgs2=wl.reorth,
                     block=max(1, min(getattr(wl, "block_actions", 1), 1 + wl.max_iter)))
    sm = caks_smoother(ssm, tr, mr) if smoother else None
    return ssm, tr, sm
