"""Synthetic workloads shaped like the paper's experiments (inputs only).

Readings (DESIGN.md §3 lists them all):
  * R13/R14 — ERA5-shaped sphere grids: a 1440x721 0.25-degree lat/lon grid
    downsampled by a factor f along both axes (Sec. 6.3
    "downsample the dataset by factors of 3, 6, 12, and 24"); the test set is the
    regular 25% subgrid {lat idx 2,4,...,n_lat-3} x {even lon idx}
    (PAPER.md:709).  This reproduces every row of Table C.1.
  * R11/R12 — points are embedded in R^3 on the unit sphere (extrinsic kernel,
    PAPER.md:2124); the spatial lengthscale is the grid spacing at the equator,
    ell_x = 0.25 f degrees in radians.
  * R15 — ERA5 values are unavailable; a deterministic "temperature-like" field
    plus N(0, lambda^2) noise (PCG64) stands in for them.  Hyperparameters follow
    App. C.2.3: ell_t = 3 h, sigma = 10, lambda = 0.1, dt = 1 h.
  * cfg1 — the 1-D exactness case of BASELINE.json configs[0]: 32 points
    x_j = 0.25 j, ell_t = ell_x = 0.5, sigma = 1, lambda = 0.1 (App. C.2.1,
    PAPER.md:2022-2032), dt = 0.05, T = 50, observed values sin(x) exp(-t) + noise
    (the toy target of PAPER.md:586, Sec. 6.2).
  * R8 — time origin t_0 = t_1: the first predict has dt = 0.

Nothing in this module evaluates a covariance kernel, an SDE or a filter.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Optional

import numpy as np

__all__ = [
    "Workload",
    "grid_1d",
    "sphere_grid",
    "era5_test_mask",
    "temperature_field",
    "farthest_point_order",
    "make_workload",
    "WORKLOADS",
]


@dataclasses.dataclass
class Workload:
    """All inputs of one CAKF/CAKS run.

    State ordering is derivative-major (Lemma B.1):
    u = (f_0(t, X); f_1(t, X); ...), D = d_time * n_space.
    """

    name: str
    coords: np.ndarray            # (N_X, space_dim) float64, already embedded
    times: np.ndarray             # (T,) observation times t_1..t_T
    dts: np.ndarray               # (T,) dt of the predict INTO step k (dts[0] = 0, R8)
    obs_idx: list                 # per step: int64 spatial indices (empty = IsMissing)
    y: list                       # per step: float64 observed values
    noise_var: list               # per step: float64 diag(Lambda_k)
    test_idx: np.ndarray          # spatial indices never observed
    d_time: int = 2               # D' (2 = Matern-3/2 temporal prior)
    nu_t: float = 1.5
    ell_t: float = 0.5
    sigma: float = 1.0            # temporal output scale (Sigma^t = sigma^2 Matern)
    nu_x: float = 1.5
    ell_x: float = 0.5            # spatial lengthscale (coordinate units)
    lam: float = 0.1              # observation noise std (Lambda = lam^2 I)
    policy: str = "cg"            # "cg" | "coord" | "random"
    max_iter: int = 64            # N^max per step
    max_rank: int = -1            # r cap; < 0 = never truncate
    coord_order: Optional[list] = None  # per step: int64 positions into obs_idx (coord policy)
    action_seed: int = 1          # Philox key for the random policy (R16)
    rtol: float = 0.0
    reorth: bool = True           # second Gram-Schmidt pass (CGS2, reading R19)
    block_actions: int = 1      # block execution of non-adaptive policies (b actions per K2 product)

    @property
    def n_space(self) -> int:
        return int(self.coords.shape[0])

    @property
    def space_dim(self) -> int:
        return int(self.coords.shape[1])

    @property
    def D(self) -> int:
        return self.d_time * self.n_space

    @property
    def T(self) -> int:
        return len(self.times)

    def n_obs(self, k: int) -> int:
        """Observations at step k = 1..T."""
        return int(len(self.obs_idx[k - 1]))

    def summary(self) -> dict:
        return {
            "workload": self.name,
            "N_X": self.n_space,
            "D": self.D,
            "N": self.n_obs(1) if self.T else 0,
            "T": self.T,
            "policy": self.policy,
            "max_iter": self.max_iter,
            "max_rank": self.max_rank,
        }


def grid_1d(n: int, spacing: float) -> np.ndarray:
    """x_j = spacing * j, j = 0..n-1, as an (n, 1) array."""
    return (spacing * np.arange(n, dtype=np.float64))[:, None]


def sphere_grid(n_lon: int, n_lat: int, step_deg: float):
    """Regular lat/lon grid embedded on the unit sphere in R^3 (lat-major order).

    lon_j = step*j, lat_i = 90 - step*i (R14).  Pole rows collapse to one R^3
    point each (duplicates are kept, as in the gridded data).
    Returns (xyz (n_lat*n_lon, 3), lat_rad, lon_rad) with lat/lon per point.
    """
    lon = np.deg2rad(step_deg * np.arange(n_lon, dtype=np.float64))
    lat = np.deg2rad(90.0 - step_deg * np.arange(n_lat, dtype=np.float64))
    LAT, LON = np.meshgrid(lat, lon, indexing="ij")
    LAT = LAT.ravel()
    LON = LON.ravel()
    xyz = np.stack([np.cos(LAT) * np.cos(LON), np.cos(LAT) * np.sin(LON), np.sin(LAT)], axis=1)
    return xyz, LAT, LON


def era5_test_mask(n_lon: int, n_lat: int) -> np.ndarray:
    """Boolean mask (lat-major) of the 25% regular test subgrid (R13)."""
    li = np.arange(n_lat)
    lj = np.arange(n_lon)
    lat_ok = (li >= 2) & (li <= n_lat - 3) & (li % 2 == 0)
    lon_ok = lj % 2 == 0
    return (lat_ok[:, None] & lon_ok[None, :]).ravel()


def temperature_field(t_hours, lat, lon) -> np.ndarray:
    """Deterministic 'temperature-like' field in deg C (R15)."""
    return (
        15.0
        - 40.0 * np.sin(lat) ** 2
        + 8.0 * np.cos(lat) * np.cos(lon - 2.0 * np.pi * t_hours / 24.0)
        + 3.0 * np.sin(3.0 * lon) * np.cos(2.0 * lat)
    )


def farthest_point_order(points: np.ndarray, n: int) -> np.ndarray:
    """Greedy farthest-point order over `points` (lowest index breaks ties) (R17).

    A space-filling order for the coordinate policy (App. C.3).
    """
    n = min(n, len(points))
    order = np.empty(n, dtype=np.int64)
    d2 = np.full(len(points), np.inf)
    cur = 0
    for i in range(n):
        order[i] = cur
        d2 = np.minimum(d2, np.sum((points - points[cur]) ** 2, axis=1))
        d2[order[: i + 1]] = -1.0
        cur = int(np.argmax(d2))
    return order


def _sphere_workload(name, factor=None, n_lon=None, n_lat=None, step_deg=None, T=48,
                     policy="cg", max_iter=64, max_rank=256, seed=0, **kw) -> Workload:
    if factor is not None:
        n_lon, n_lat, step_deg = 1440 // factor, 720 // factor + 1, 0.25 * factor
    xyz, lat, lon = sphere_grid(n_lon, n_lat, step_deg)
    test = era5_test_mask(n_lon, n_lat)
    train_idx = np.flatnonzero(~test).astype(np.int64)
    test_idx = np.flatnonzero(test).astype(np.int64)
    times = np.arange(T, dtype=np.float64)  # hours
    dts = np.concatenate([[0.0], np.diff(times)])
    rng = np.random.Generator(np.random.PCG64(seed))
    lam = 0.1
    ys, idxs, nvs = [], [], []
    for k in range(T):
        f = temperature_field(times[k], lat[train_idx], lon[train_idx])
        ys.append(f + lam * rng.standard_normal(len(train_idx)))
        idxs.append(train_idx.copy())
        nvs.append(np.full(len(train_idx), lam * lam))
    ell_x = np.deg2rad(step_deg)  # R12: grid spacing at the equator (unit sphere)
    wl = Workload(name=name, coords=xyz, times=times, dts=dts, obs_idx=idxs, y=ys,
                  noise_var=nvs, test_idx=test_idx, d_time=2, nu_t=1.5, ell_t=3.0,
                  sigma=10.0, nu_x=1.5, ell_x=float(ell_x), lam=lam, policy=policy,
                  max_iter=max_iter, max_rank=max_rank)
    for key, val in kw.items():
        setattr(wl, key, val)
    if wl.policy == "coord" and wl.coord_order is None:
        pts = xyz[train_idx]
        order = farthest_point_order(pts, wl.max_iter)
        wl.coord_order = [order.copy() for _ in range(T)]
    return wl


def _line_workload(name, n=32, spacing=0.25, T=50, dt=0.05, test_every=4, test_offset=3,
                   policy="coord", max_iter=None, max_rank=-1, seed=0, lam=0.1,
                   ell=0.5, sigma=1.0, **kw) -> Workload:
    coords = grid_1d(n, spacing)
    test = np.zeros(n, dtype=bool)
    if test_every:
        test[test_offset::test_every] = True
    train_idx = np.flatnonzero(~test).astype(np.int64)
    test_idx = np.flatnonzero(test).astype(np.int64)
    times = dt * np.arange(T, dtype=np.float64)
    dts = np.concatenate([[0.0], np.diff(times)])
    rng = np.random.Generator(np.random.PCG64(seed))
    ys, idxs, nvs = [], [], []
    for k in range(T):
        x = coords[train_idx, 0]
        ys.append(np.sin(x) * np.exp(-times[k]) + lam * rng.standard_normal(len(train_idx)))
        idxs.append(train_idx.copy())
        nvs.append(np.full(len(train_idx), lam * lam))
    N = len(train_idx)
    mi = N if max_iter is None else max_iter
    wl = Workload(name=name, coords=coords, times=times, dts=dts, obs_idx=idxs, y=ys,
                  noise_var=nvs, test_idx=test_idx, d_time=2, nu_t=1.5, ell_t=ell,
                  sigma=sigma, nu_x=1.5, ell_x=ell, lam=lam, policy=policy, max_iter=mi,
                  max_rank=max_rank)
    for key, val in kw.items():
        setattr(wl, key, val)
    if wl.policy == "coord" and wl.coord_order is None:
        wl.coord_order = [np.arange(min(N, wl.max_iter), dtype=np.int64) for _ in range(T)]
    return wl


WORKLOADS: dict = {
    # BASELINE.json configs[0]: D = 64 exactness case (full-rank unit-vector actions, no truncation)
    "cfg1": lambda **kw: _line_workload("cfg1", **kw),
    # BASELINE.json configs[1]: D = 14,640 (ERA5 / 12)
    "cfg2": lambda **kw: _sphere_workload("cfg2", factor=12, **{"max_rank": 256, **kw}),
    # BASELINE.json configs[2]: D = 231,360 (ERA5 / 3)
    "cfg3": lambda **kw: _sphere_workload("cfg3", factor=3, **{"max_rank": 512, **kw}),
    # BASELINE.json configs[3]: D ~ 1.0M, 0.36 degree grid (R14 proposal)
    "cfg4": lambda **kw: _sphere_workload("cfg4", n_lon=1000, n_lat=501, step_deg=0.36,
                                          **{"T": 24, "max_rank": 1024, **kw}),
    # parity-test sizes (span several tiles plus a ragged tail; dense oracle runs in seconds)
    "sphere48": lambda **kw: _sphere_workload("sphere48", factor=48,
                                              **{"T": 6, "max_iter": 16, "max_rank": 24, **kw}),
    "sphere24": lambda **kw: _sphere_workload("sphere24", factor=24,
                                              **{"T": 5, "max_iter": 24, "max_rank": 40, **kw}),
    "line8": lambda **kw: _line_workload("line8", **{"n": 8, "T": 4, "test_every": 4,
                                                     "test_offset": 1, **kw}),
}


def make_workload(name: str, **overrides) -> Workload:
    """Build a named workload; keyword overrides replace Workload fields or builder args."""
    if name not in WORKLOADS:
        raise KeyError(f"unknown workload {name!r}; known: {sorted(WORKLOADS)}")
    return WORKLOADS[name](**overrides)
