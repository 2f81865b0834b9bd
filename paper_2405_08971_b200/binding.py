"""Thin ctypes binding of libcakf.so — argument marshalling only.

Every step of the CAKF/CAKS path runs in libcakf's CUDA kernels; this module only
converts Python / numpy / torch arguments into the C-ABI of ``include/cakf.h``
(same function names).  There is no CPU fallback: if the shared library or a CUDA
device is missing, calls raise ``CakfError``.

Arrays may be numpy arrays (host) or CUDA torch tensors (device); the library
copies either kind (UVA).  Torch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CAKF_LIB") or os.path.join(HERE, "libcakf.so")   # CAKF_LIB: experiment builds

CAKF_F32, CAKF_F64 = 0, 1
CAKF_MATERN12, CAKF_MATERN32, CAKF_MATERN52 = 1, 3, 5
CAKF_POLICY_CG, CAKF_POLICY_COORD, CAKF_POLICY_RANDOM, CAKF_POLICY_BLOCKRES = 0, 1, 2, 3
CAKF_PRED, CAKF_FILTER, CAKF_SMOOTH = 0, 1, 2
POLICIES = {"cg": CAKF_POLICY_CG, "coord": CAKF_POLICY_COORD, "random": CAKF_POLICY_RANDOM,
            "blockres": CAKF_POLICY_BLOCKRES}
KERNELS = {0.5: CAKF_MATERN12, 1.5: CAKF_MATERN32, 2.5: CAKF_MATERN52}
DTYPES = {"f32": CAKF_F32, "f64": CAKF_F64, np.float32: CAKF_F32, np.float64: CAKF_F64}


class CakfError(RuntimeError):
    pass


class cakf_config(ctypes.Structure):
    _fields_ = [
        ("dtype", ctypes.c_int32), ("d_time", ctypes.c_int32), ("n_space", ctypes.c_int64),
        ("space_dim", ctypes.c_int32), ("coords", ctypes.c_void_p), ("spatial_kernel", ctypes.c_int32),
        ("ell_x", ctypes.c_double), ("sigma_t0", ctypes.c_void_p), ("mu0", ctypes.c_void_p),
        ("policy", ctypes.c_int32), ("max_iter", ctypes.c_int32), ("max_rank", ctypes.c_int32),
        ("rtol", ctypes.c_double), ("reorth", ctypes.c_int32), ("cull_zero", ctypes.c_int32), ("block_actions", ctypes.c_int32), ("keep_carriers", ctypes.c_int32), ("seed", ctypes.c_uint64), ("max_steps", ctypes.c_int32),
        ("max_obs", ctypes.c_int64), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
        ("nccl_id", ctypes.c_void_p), ("stream", ctypes.c_void_p),
    ]


class cakf_step_stats(ctypes.Structure):
    _fields_ = [
        ("k", ctypes.c_int32), ("iters", ctypes.c_int32), ("rejected", ctypes.c_int32),
        ("rank_in", ctypes.c_int32), ("cols", ctypes.c_int32), ("rank_out", ctypes.c_int32),
        ("smoother_rank", ctypes.c_int32), ("missing", ctypes.c_int32), ("res0", ctypes.c_double),
        ("res_final", ctypes.c_double), ("eta_min", ctypes.c_double), ("dropped_mass", ctypes.c_double),
    ]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


EXPORTS = [
    "cakf_create", "cakf_reset", "cakf_predict", "cakf_update", "cakf_truncate", "caks_smooth", "cakf_get",
    "cakf_get_stats", "cakf_get_kept_eigs", "cakf_sync", "cakf_destroy", "cakf_last_error", "cakf_version",
    "cakf_matern_transition", "cakf_gram_matmul", "cakf_profile", "cakf_profile_read", "cakf_kernel_launches",
    "cakf_nccl_unique_id", "cakf_shard_plan", "cakf_sym_unit_blocks", "cakf_cull_stats", "cakf_interpolate", "cakf_sample",
    "cakf_lowrank_gemm", "cakf_debug_matvec", "cakf_sym_eig", "cakf_alu_peaks",
]
PROF_CATEGORIES = ["k1_matvec", "k2_post", "k2_smooth", "loop_stages", "truncate", "lowrank", "trunc_gram",
                   "trunc_eig", "trunc_gemm"]

_lib = None


def load(path: str = LIB_PATH):
    """Load libcakf.so (raises CakfError if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise CakfError(f"{path} not built: run `python -m paper_2405_08971_b200.build`")
    lib = ctypes.CDLL(path)
    vp, i32, i64, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    lib.cakf_create.argtypes = [ctypes.POINTER(cakf_config), ctypes.POINTER(vp)]
    lib.cakf_reset.argtypes = [vp]
    lib.cakf_predict.argtypes = [vp, vp, vp, vp]
    lib.cakf_update.argtypes = [vp, i64, vp, vp, vp, vp]
    lib.cakf_truncate.argtypes = [vp]
    lib.caks_smooth.argtypes = [vp]
    lib.cakf_get.argtypes = [vp, i32, i32, vp, vp]
    lib.cakf_get_stats.argtypes = [vp, i32, ctypes.POINTER(cakf_step_stats)]
    lib.cakf_get_kept_eigs.argtypes = [vp, i32, vp, i32, ctypes.POINTER(i32)]
    lib.cakf_sync.argtypes = [vp]
    lib.cakf_destroy.argtypes = [vp]
    lib.cakf_last_error.restype = ctypes.c_char_p
    lib.cakf_matern_transition.argtypes = [i32, f64, f64, f64, vp, vp, vp]
    lib.cakf_gram_matmul.argtypes = [i32, i32, f64, i32, i64, vp, i64, vp, i32, vp, f64, vp, vp]
    lib.cakf_lowrank_gemm.argtypes = [i32, i32, i64, i64, i64, f64, vp, i64, vp, i64, f64, vp, i64, vp]
    lib.cakf_profile.argtypes = [vp, i32]
    lib.cakf_profile_read.argtypes = [vp, vp, vp, i32]
    lib.cakf_kernel_launches.restype = ctypes.c_int64
    lib.cakf_nccl_unique_id.argtypes = [vp]
    lib.cakf_shard_plan.argtypes = [i64, i64, i32, i32, vp]
    lib.cakf_cull_stats.argtypes = [vp, vp]
    lib.cakf_debug_matvec.argtypes = [vp, i64, vp, vp, vp, i32]
    lib.cakf_sym_eig.argtypes = [i64, i64, vp, vp, vp, vp]
    lib.cakf_alu_peaks.argtypes = [vp, vp]
    lib.cakf_interpolate.argtypes = [vp, i32, vp, vp, vp, i32, vp, vp]
    lib.cakf_sample.argtypes = [vp, i32, vp, vp, vp, i32, vp]
    lib.cakf_sym_unit_blocks.argtypes = [i64, i64, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    for name in EXPORTS:
        if name not in ("cakf_last_error", "cakf_version", "cakf_kernel_launches"):
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _check(rc: int):
    if rc != 0:
        msg = load().cakf_last_error().decode(errors="replace")
        raise CakfError(f"libcakf status {rc}: {msg}")


def _ptr(x):
    """(pointer, keepalive) for numpy / torch / None."""
    if x is None:
        return None, None
    if hasattr(x, "data_ptr"):  # torch tensor
        if not x.is_contiguous():
            x = x.contiguous()
        return x.data_ptr(), x
    a = np.ascontiguousarray(x)
    return a.ctypes.data, a


def kernel_launches() -> int:
    """Number of libcakf kernels launched by this process so far."""
    return int(load().cakf_kernel_launches())


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (create on rank 0, broadcast, pass as nccl_id)."""
    buf = ctypes.create_string_buffer(128)
    _check(load().cakf_nccl_unique_id(buf))
    return buf.raw


def shard_plan(n_space: int, n_obs: int, world: int, rank: int) -> dict:
    """Rows of the K2 output and units of the symmetric K1 owned by `rank` (host-only)."""
    out = np.zeros(7, dtype=np.int64)
    _check(load().cakf_shard_plan(int(n_space), int(n_obs), int(world), int(rank), out.ctypes.data))
    return dict(zip(["row_lo", "row_hi", "u_lo", "u_hi", "n_units", "slice_rows", "block_points"],
                    (int(v) for v in out)))


def sym_unit_blocks(n_obs: int, unit: int):
    """(bi, bj) tile blocks of a symmetric K1 unit (host mirror of the device map)."""
    bi, bj = ctypes.c_int32(0), ctypes.c_int32(0)
    _check(load().cakf_sym_unit_blocks(int(n_obs), int(unit), ctypes.byref(bi), ctypes.byref(bj)))
    return bi.value, bj.value


def matern_transition(nu: float, ell_t: float, sigma: float, dt: float):
    """(A^t(dt), Q^t(dt), Sigma_inf) from the library's closed forms (R10)."""
    lib = load()
    nu2 = int(round(2 * nu))
    n = (nu2 + 1) // 2
    A = np.zeros((n, n))
    Q = np.zeros((n, n))
    S = np.zeros((n, n))
    _check(lib.cakf_matern_transition(nu2, float(ell_t), float(sigma), float(dt), A.ctypes.data, Q.ctypes.data,
                                      S.ctypes.data))
    return A, Q, S


def gram_matmul(xr, xc, X, nu: float, ell: float, alpha: float = 1.0, out=None, stream=None):
    """Y = alpha * K(xr, xc) X on the device (torch CUDA tensors, dtype f32/f64)."""
    import torch
    lib = load()
    dtype = CAKF_F32 if xr.dtype == torch.float32 else CAKF_F64
    n_rhs = 1 if X.dim() == 1 else X.shape[1]
    Xc = X.reshape(-1, n_rhs).t().contiguous()  # column-major n_cols x n_rhs
    Y = torch.empty((n_rhs, xr.shape[0]), dtype=xr.dtype, device=xr.device)
    _check(lib.cakf_gram_matmul(dtype, KERNELS[nu], float(ell), xr.shape[1], xr.shape[0], xr.contiguous().data_ptr(),
                                xc.shape[0], xc.contiguous().data_ptr(), n_rhs, Xc.data_ptr(), float(alpha),
                                Y.data_ptr(), stream))
    Y = Y.t()
    return Y[:, 0] if X.dim() == 1 else Y


def lowrank_gemm(A, B, transa=False, transb=False, alpha=1.0, beta=0.0, C=None, stream=None):
    """alpha op(A) @ op(B) + beta C for fp32 CUDA tensors (fp64-accurate, INT8 tensor cores).

    torch tensors are row-major; a row-major (r, c) tensor is the column-major (c, r) matrix, so
    the call computes C^T = op(B)^T op(A)^T in the library's column-major convention."""
    import torch
    lib = load()
    Am, Bm = A.contiguous(), B.contiguous()
    m = Am.shape[1] if transa else Am.shape[0]
    k = Am.shape[0] if transa else Am.shape[1]
    n = Bm.shape[0] if transb else Bm.shape[1]
    out = torch.zeros((m, n), dtype=torch.float32, device=A.device) if C is None else C
    assert out.is_contiguous() and out.shape == (m, n) and out.dtype == torch.float32
    _check(lib.cakf_lowrank_gemm(1 if transb else 0, 1 if transa else 0, n, m, k, float(alpha),
                                 Bm.data_ptr(), Bm.shape[1], Am.data_ptr(), Am.shape[1], float(beta),
                                 out.data_ptr(), n, stream))
    return out


def alu_peaks(stream=None) -> dict:
    """Live microbenchmarks (cakf_alu_peaks): MUFU ops/s and fp64 tensor-core flop/s."""
    out = np.zeros(3)
    _check(load().cakf_alu_peaks(out.ctypes.data, stream))
    return {"mufu_ops_per_s": float(out[0]), "dmma_flop_per_s": float(out[1])}


def sym_eig(G, r=None):
    """(w ascending, Qr (c x r) eigenvectors of the r largest eigenvalues, descending) of a symmetric fp64
    matrix through the library's device eigensolver (cakf_sym_eig); numpy in / out."""
    Gf = np.asfortranarray(np.asarray(G, dtype=np.float64))
    c = Gf.shape[0]
    r = c if r is None else int(r)
    w = np.empty(c)
    Q = np.empty((c, max(r, 1)), order="F")
    _check(load().cakf_sym_eig(c, r, Gf.ctypes.data, w.ctypes.data, Q.ctypes.data, None))
    return w, Q[:, :r]


class Cakf:
    """One CAKF/CAKS handle (``cakf_t``).  Methods map 1:1 onto the C-ABI."""

    def __init__(self, coords, ell_x, sigma_t0, *, dtype="f32", d_time=2, nu_x=1.5, mu0=None, policy="cg",
                 max_iter=64, max_rank=-1, seed=1, max_steps=48, max_obs=0, reorth=True, stream=None,
                 rank=0, world=1, nccl_id=None, cull_zero=True, keep_carriers=False, block_actions=1):
        self.lib = load()
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        if coords.ndim == 1:
            coords = coords[:, None]
        self.np_dtype = np.float32 if DTYPES[dtype] == CAKF_F32 else np.float64
        self.n_space, self.space_dim = coords.shape
        self.d_time = d_time
        self.D = d_time * self.n_space
        st0 = np.ascontiguousarray(sigma_t0, dtype=np.float64)
        mu = None if mu0 is None else np.ascontiguousarray(mu0, dtype=np.float64)
        cfg = cakf_config(dtype=DTYPES[dtype], d_time=d_time, n_space=self.n_space, space_dim=self.space_dim,
                          coords=coords.ctypes.data, spatial_kernel=KERNELS[nu_x], ell_x=float(ell_x),
                          sigma_t0=st0.ctypes.data, mu0=None if mu is None else mu.ctypes.data,
                          policy=POLICIES[policy] if isinstance(policy, str) else int(policy),
                          max_iter=int(max_iter), max_rank=int(max_rank), rtol=0.0, reorth=int(bool(reorth)),
                          cull_zero=int(bool(cull_zero)), keep_carriers=int(bool(keep_carriers)), block_actions=int(block_actions),
                          seed=int(seed),
                          max_steps=int(max_steps), max_obs=int(max_obs), rank=int(rank), world=int(world),
                          nccl_id=None, stream=stream)
        self._nccl_id = None
        if world > 1:
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            cfg.nccl_id = ctypes.cast(self._nccl_id, ctypes.c_void_p)
        h = ctypes.c_void_p()
        _check(self.lib.cakf_create(ctypes.byref(cfg), ctypes.byref(h)))
        self.h = h

    # --- the C-ABI, 1:1
    def reset(self):
        _check(self.lib.cakf_reset(self.h))

    def predict(self, A_t, Q_t, b=None):
        A = np.ascontiguousarray(A_t, dtype=np.float64)
        Q = np.ascontiguousarray(Q_t, dtype=np.float64)
        pb, kb = _ptr(b)
        _check(self.lib.cakf_predict(self.h, A.ctypes.data, Q.ctypes.data, pb))

    def update(self, obs_idx, y, noise_var, coord_order=None):
        n = 0 if obs_idx is None else int(len(obs_idx))
        if n == 0:
            _check(self.lib.cakf_update(self.h, 0, None, None, None, None))
            return
        pi, ki = _ptr(obs_idx if hasattr(obs_idx, "data_ptr") else np.asarray(obs_idx, dtype=np.int64))
        py, ky = _ptr(y if hasattr(y, "data_ptr") else np.asarray(y, dtype=self.np_dtype))
        pn, kn = _ptr(noise_var if hasattr(noise_var, "data_ptr") else np.asarray(noise_var, dtype=self.np_dtype))
        po, ko = _ptr(None if coord_order is None else (coord_order if hasattr(coord_order, "data_ptr")
                                                        else np.asarray(coord_order, dtype=np.int64)))
        _check(self.lib.cakf_update(self.h, n, pi, py, pn, po))

    def truncate(self):
        _check(self.lib.cakf_truncate(self.h))

    def smooth(self):
        _check(self.lib.caks_smooth(self.h))

    def get(self, k: int, which: int = CAKF_FILTER, mean=None, var=None):
        """Returns (mean, var); numpy arrays unless device buffers are passed in."""
        if mean is None and var is None:
            mean = np.empty(self.D, dtype=self.np_dtype)
            var = np.empty(self.D, dtype=self.np_dtype)
        pm, km = _ptr(mean)
        pv, kv = _ptr(var)
        _check(self.lib.cakf_get(self.h, int(k), int(which), pm, pv))
        return mean, var

    def get_stats(self, k: int) -> dict:
        s = cakf_step_stats()
        _check(self.lib.cakf_get_stats(self.h, int(k), ctypes.byref(s)))
        return s.as_dict()

    def get_kept_eigs(self, k: int, cap: int = 4096) -> np.ndarray:
        vals = np.zeros(cap)
        n = ctypes.c_int32(0)
        _check(self.lib.cakf_get_kept_eigs(self.h, int(k), vals.ctypes.data, cap, ctypes.byref(n)))
        return vals[: n.value].copy()

    def sync(self):
        _check(self.lib.cakf_sync(self.h))

    def profile(self, enable: bool = True):
        _check(self.lib.cakf_profile(self.h, int(bool(enable))))

    def profile_read(self, reset: bool = True) -> dict:
        """{category: (total_ms, launches)} of the launches recorded since the last reset."""
        n = len(PROF_CATEGORIES)
        ms = np.zeros(n)
        cnt = np.zeros(n, dtype=np.int64)
        _check(self.lib.cakf_profile_read(self.h, ms.ctypes.data, cnt.ctypes.data, int(bool(reset))))
        return {c: (float(ms[i]), int(cnt[i])) for i, c in enumerate(PROF_CATEGORIES)}

    def interpolate(self, k: int, A1, Q1, A2=None, which: int = CAKF_SMOOTH):
        """Mean and variance (numpy, user point order) at t in [t_k, t_{k+1}) (cakf_interpolate)."""
        a1 = np.ascontiguousarray(A1, dtype=np.float64)
        q1 = np.ascontiguousarray(Q1, dtype=np.float64)
        a2 = None if A2 is None else np.ascontiguousarray(A2, dtype=np.float64)
        mean = np.empty(self.D, dtype=self.np_dtype)
        var = np.empty(self.D, dtype=self.np_dtype)
        _check(self.lib.cakf_interpolate(self.h, int(k), a1.ctypes.data, q1.ctypes.data,
                                         None if a2 is None else a2.ctypes.data, int(which),
                                         mean.ctypes.data, var.ctypes.data))
        return mean, var

    def sample(self, x0, q, eps, which: int = CAKF_SMOOTH) -> np.ndarray:
        """Posterior samples (cakf_sample).  x0: D x S; q: list of T arrays D x S; eps: list of
        N_k x S arrays for the non-missing steps.  Returns (T+1) x D x S (numpy, user order)."""
        x0 = np.asarray(x0, dtype=self.np_dtype)
        if x0.ndim == 1:
            x0 = x0[:, None]
        S = x0.shape[1]
        x0f = np.asfortranarray(x0)
        qf = np.concatenate([np.asfortranarray(np.asarray(a, dtype=self.np_dtype).reshape(self.D, S)).ravel(order="F")
                             for a in q])
        ef = np.concatenate([np.asfortranarray(np.asarray(a, dtype=self.np_dtype).reshape(-1, S)).ravel(order="F")
                             for a in eps] or [np.zeros(1, dtype=self.np_dtype)])
        T = len(q)
        out = np.empty((T + 1) * self.D * S, dtype=self.np_dtype)
        _check(self.lib.cakf_sample(self.h, int(S), x0f.ctypes.data, qf.ctypes.data, ef.ctypes.data, int(which),
                                    out.ctypes.data))
        return out.reshape(T + 1, S, self.D).transpose(0, 2, 1)

    def debug_matvec(self, obs_idx, s, shares=1):
        """K(X_obs, X_obs) s through the inner loop's own K1 launch path (cakf_debug_matvec); numpy in/out.
        shares > 1: K1 as the multi-GPU split of `shares` ranks, run one share after the other."""
        idx = np.ascontiguousarray(obs_idx, dtype=np.int64)
        sv = np.ascontiguousarray(s, dtype=self.np_dtype)
        out = np.empty(len(idx), dtype=self.np_dtype)
        _check(self.lib.cakf_debug_matvec(self.h, len(idx), idx.ctypes.data, sv.ctypes.data, out.ctypes.data,
                                          int(shares)))
        return out

    def cull_stats(self) -> dict:
        """Fractions of the dense kernel work evaluated under exact-zero culling (1.0 = none culled)."""
        out = np.zeros(3)
        _check(self.lib.cakf_cull_stats(self.h, out.ctypes.data))
        return {"k1_matvec": float(out[0]), "k2_post": float(out[1]), "k2_smooth": float(out[2])}

    def destroy(self):
        if getattr(self, "h", None):
            self.lib.cakf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass
