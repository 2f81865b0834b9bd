"""Multi-GPU decomposition on CPU: the library's shard plan (host-only C-ABI functions)
and world_size 2 / 3 gloo runs of the row-sharded exchange pattern of the device path (include/cakf.h):
rank p owns points [row_lo, row_hi) and their rows of every D-length array; [H m^-, H M^-] and K1's
N-vector (symmetric units [u_lo, u_hi)) are all-reduced, the truncation Gram is the all-reduced sum of
partial Grams (eig replicated), the smoother all-reduces M^-T x and V^T H y, K2 and the rest stay local.
The per-rank products come from the oracle, so the test checks the plan and the collectives, not the
CUDA kernels (tests/test_gpu_*: the forced-collective path at world 1, K1's balanced split emulated)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mfree
from paper_2405_08971_b200 import binding


@pytest.fixture(scope="module", autouse=True)
def lib():
    from paper_2405_08971_b200 import build
    build.build()
    binding.load()


@pytest.mark.parametrize("n_space,n_obs", [(1, 1), (1000, 700), (7320, 5580), (115680, 87120), (129, 128)])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_plan_covers_everything_once(n_space, n_obs, world):
    plans = [binding.shard_plan(n_space, n_obs, world, r) for r in range(world)]
    rows = np.zeros(n_space, dtype=int)
    units = np.zeros(plans[0]["n_units"], dtype=int)
    for p in plans:
        assert p["slice_rows"] % 128 == 0
        rows[p["row_lo"]:p["row_hi"]] += 1
        units[p["u_lo"]:p["u_hi"]] += 1
    assert np.all(rows == 1) and np.all(units == 1)


@pytest.mark.parametrize("n_obs", [1, 1024, 1025, 5580, 87120])
def test_sym_units_enumerate_block_pairs_once(n_obs):
    plan = binding.shard_plan(1, n_obs, 1, 0)
    bp = plan["block_points"]
    assert bp % 128 == 0
    nb = (n_obs + bp - 1) // bp
    U = plan["n_units"]
    assert U == nb * (nb + 1) // 2
    seen = set()
    for u in range(U):
        bi, bj = binding.sym_unit_blocks(n_obs, u)
        assert 0 <= bi <= bj < nb
        seen.add((bi, bj))
    assert len(seen) == U


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, prob, out_q):
    """One rank of the row-sharded exchange pattern of the device path (include/cakf.h, multi-GPU):
    rows [row_lo, row_hi) of every D-length array (both derivative blocks), replicated N-length state."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    binding.load()
    X, s, M, x, V, obs, nu, ell, Dp, r = (prob[k] for k in ("X", "s", "M", "x", "V", "obs", "nu", "ell", "Dp", "r"))
    NX = len(X)
    plan = binding.shard_plan(NX, len(obs), world, rank)
    lo, hi = plan["row_lo"], plan["row_hi"]
    rows = np.concatenate([np.arange(lo, hi) + d * NX for d in range(Dp)])   # this rank's D rows
    Mp, xp = M[rows], x[rows]

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t)
        return t.numpy()

    out = {}
    # update: [H m^-, H M^-] -- each rank the observed rows it owns, zeros elsewhere, summed
    own = (obs >= lo) & (obs < hi)
    HMp = np.zeros((len(obs), M.shape[1]))
    HMp[own] = M[obs[own]]
    out["HM"] = allreduce(HMp)
    # K1: this rank's symmetric units (index split of the plan), all-reduce of the N-vector
    Xt = X[obs]
    n = len(obs)
    y = np.zeros(n)
    bp = plan["block_points"]
    for u in range(plan["u_lo"], plan["u_hi"]):
        bi, bj = binding.sym_unit_blocks(n, u)
        I = slice(bi * bp, min(n, (bi + 1) * bp))
        J = slice(bj * bp, min(n, (bj + 1) * bp))
        if bi == bj:
            y[I] += mfree.gram_apply(Xt[I], Xt[I], s[I], nu, ell)
        else:
            y[I] += mfree.gram_apply(Xt[I], Xt[J], s[J], nu, ell)
            y[J] += mfree.gram_apply(Xt[J], Xt[I], s[I], nu, ell)
    out["Ks"] = allreduce(y)
    # post-loop K2: this rank's rows of K(X, X_T) [v V] -- no exchange
    out["KV_rows"] = (lo, hi, mfree.gram_apply(X[lo:hi], Xt, V, nu, ell))
    # truncation: partial Grams summed, replicated eig, local rows of M Q_r
    G = allreduce(Mp.T @ Mp)
    lam, Q = np.linalg.eigh(G)
    out["G"] = G
    out["MQ_rows"] = (rows, Mp @ Q[:, -r:])
    # smoother: M^T x partials summed, local rows of y = x - M (M^T x); V^T H y partial over owned observations
    t = allreduce(Mp.T @ xp)
    yl = xp - Mp @ t
    out["y_rows"] = (rows, yl)
    Hy = np.zeros((n, x.shape[1]))
    pos = {g: i for i, g in enumerate(rows)}
    for j, o in enumerate(obs):
        if lo <= o < hi:
            Hy[j] = yl[pos[o]]
    out["VtHy"] = allreduce(V.T @ Hy)
    out_q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_space,world", [(300, 2), (700, 3)])
def test_row_sharded_exchanges_gloo(n_space, world):
    """The row-sharded decomposition with the library's own plan (cakf_shard_plan), world 2 and 3 on gloo:
    every exchanged quantity equals its unsharded value, every local row block reassembles the full one."""
    rng = np.random.default_rng(n_space)
    Dp, c, r = 2, 12, 8
    X = rng.standard_normal((n_space, 3)) * 2.0
    obs = np.sort(rng.choice(n_space, n_space * 3 // 4, replace=False))
    prob = {"X": X, "s": rng.standard_normal(len(obs)), "M": rng.standard_normal((Dp * n_space, c)),
            "x": rng.standard_normal((Dp * n_space, 5)), "V": rng.standard_normal((len(obs), 4)), "obs": obs,
            "nu": 1.5, "ell": 0.9, "Dp": Dp, "r": r}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, world, port, prob, q)) for k in range(world)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    M, x, V = prob["M"], prob["x"], prob["V"]
    Xt = X[obs]
    G = M.T @ M
    lam, Q = np.linalg.eigh(G)
    y_full = x - M @ (M.T @ x)
    KV = mfree.gram_apply(X, Xt, V, 1.5, 0.9)
    MQ = M @ Q[:, -r:]
    KV_got, MQ_got, y_got = np.zeros_like(KV), np.zeros_like(MQ), np.zeros_like(y_full)
    for k, o in outs.items():
        assert np.allclose(o["HM"], M[obs], rtol=0, atol=0)             # zeros + one value: exact
        assert np.allclose(o["Ks"], mfree.gram_apply(Xt, Xt, prob["s"], 1.5, 0.9), rtol=1e-12, atol=1e-10)
        assert np.allclose(o["G"], G, rtol=1e-12, atol=1e-10)
        assert np.allclose(o["VtHy"], V.T @ y_full[obs], rtol=1e-12, atol=1e-10)
        lo, hi, blk = o["KV_rows"]
        KV_got[lo:hi] = blk
        rows, blk = o["MQ_rows"]
        MQ_got[rows] = blk
        rows, blk = o["y_rows"]
        y_got[rows] = blk
    assert np.allclose(KV_got, KV, rtol=1e-12, atol=1e-10)
    # eigenvectors: equal up to sign per column (identical Gram bits on every rank -> identical eig)
    assert np.allclose(np.abs(MQ_got), np.abs(MQ), rtol=1e-9, atol=1e-9)
    assert np.allclose(y_got, y_full, rtol=1e-12, atol=1e-10)
