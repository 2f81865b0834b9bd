"""Multi-GPU decomposition on CPU: the library's shard plan (host-only C-ABI
functions) and a world_size-2 gloo run of the same exchange pattern the GPU path uses:
  K1  rank p evaluates symmetric tile-block units [u_lo, u_hi), all-reduce(sum) of the N-vector;
  K2  rank p computes output rows [row_lo, row_hi), all-gather of the row slices.
The per-rank products here come from the oracle's chunked kernel rows, so the test checks the
plan and the collectives, not the CUDA kernels (those are covered by the GPU parity tests)."""
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


def _worker(rank, world, port, X, s, B, nu, ell, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    binding.load()
    n = len(X)
    plan = binding.shard_plan(n, n, world, rank)
    # K1: this rank's symmetric units -> partial N-vector, then all-reduce
    y = np.zeros(n)
    bp = plan["block_points"]
    for u in range(plan["u_lo"], plan["u_hi"]):
        bi, bj = binding.sym_unit_blocks(n, u)
        I = slice(bi * bp, min(n, (bi + 1) * bp))
        J = slice(bj * bp, min(n, (bj + 1) * bp))
        if bi == bj:
            y[I] += mfree.gram_apply(X[I], X[I], s[I], nu, ell)
        else:
            y[I] += mfree.gram_apply(X[I], X[J], s[J], nu, ell)
            y[J] += mfree.gram_apply(X[J], X[I], s[I], nu, ell)
    yt = torch.from_numpy(y)
    dist.all_reduce(yt)
    # K2: this rank's output row slice, then all-gather of equal-size (padded) slices
    slice_rows = plan["slice_rows"]
    Ys = np.zeros((slice_rows, B.shape[1]))
    lo, hi = plan["row_lo"], plan["row_hi"]
    if hi > lo:
        Ys[: hi - lo] = mfree.gram_apply(X[lo:hi], X, B, nu, ell)
    parts = [torch.zeros_like(torch.from_numpy(Ys)) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(Ys))
    Y = torch.cat(parts)[:n].numpy()
    if rank == 0:
        out_q.put((yt.numpy(), Y))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [300, 2100])
def test_sharded_products_gloo_world2(n):
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, 3)) * 2.0
    s = rng.standard_normal(n)
    B = rng.standard_normal((n, 5))
    nu, ell = 1.5, 0.9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, X, s, B, nu, ell, q)) for r in range(2)]
    for p in procs:
        p.start()
    y, Y = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref_y = mfree.gram_apply(X, X, s, nu, ell)
    ref_Y = mfree.gram_apply(X, X, B, nu, ell)
    assert np.allclose(y, ref_y, rtol=1e-12, atol=1e-10)
    assert np.allclose(Y, ref_Y, rtol=1e-12, atol=1e-10)
