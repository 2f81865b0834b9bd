"""Host-side call sequence of one CAKF + CAKS run through the C-ABI (alg:mfkf + alg:mfks).

    for k = 1..T:  cakf_predict(A^t_k, Q^t_k) -> cakf_update(y_k) -> cakf_truncate()
    caks_smooth()

``problem`` is any object with the fields of ``synth.Workload`` (duck-typed; this
package does not import the generators).  Inputs can be staged on the device once
(``stage_inputs``) so the timed region contains only library work, or passed as
host numpy arrays (the end-to-end path: host->device copies inside the calls).
"""
from __future__ import annotations

import numpy as np

from .binding import Cakf, matern_transition


def transitions(problem):
    """Per-step (A^t_k, Q^t_k) and Sigma_inf from the library's closed forms."""
    out = []
    Sinf = None
    for dt in problem.dts:
        A, Q, Sinf = matern_transition(problem.nu_t, problem.ell_t, problem.sigma, float(dt))
        out.append((A, Q))
    if Sinf is None:
        _, _, Sinf = matern_transition(problem.nu_t, problem.ell_t, problem.sigma, 0.0)
    return out, Sinf


def make_handle(problem, dtype="f32", stream=None, max_steps=None, rank=0, world=1, nccl_id=None, cull_zero=True,
                keep_carriers=False):
    _, Sinf = transitions(problem)
    max_obs = max((len(i) for i in problem.obs_idx), default=0)
    return Cakf(problem.coords, problem.ell_x, Sinf, dtype=dtype, d_time=problem.d_time, nu_x=problem.nu_x,
                policy=problem.policy, max_iter=problem.max_iter, max_rank=problem.max_rank,
                seed=problem.action_seed, max_steps=max_steps or problem.T, max_obs=max(max_obs, 1),
                reorth=getattr(problem, "reorth", True), stream=stream, rank=rank, world=world, nccl_id=nccl_id,
                cull_zero=cull_zero, keep_carriers=keep_carriers,
                block_actions=getattr(problem, "block_actions", 1))


def stage_inputs(problem, dtype="f32", device="cuda"):
    """Per-step inputs as device torch tensors (idx int64, y, noise_var, coord order)."""
    import torch
    tdt = torch.float32 if dtype == "f32" else torch.float64
    steps = []
    for k in range(problem.T):
        idx = torch.as_tensor(np.asarray(problem.obs_idx[k], dtype=np.int64), device=device)
        y = torch.as_tensor(np.asarray(problem.y[k]), dtype=tdt, device=device)
        nv = torch.as_tensor(np.asarray(problem.noise_var[k]), dtype=tdt, device=device)
        order = None
        if problem.policy == "coord" and problem.coord_order is not None:
            order = torch.as_tensor(np.asarray(problem.coord_order[k], dtype=np.int64), device=device)
        steps.append((idx, y, nv, order))
    return steps


def host_inputs(problem, dtype="f32"):
    npdt = np.float32 if dtype == "f32" else np.float64
    steps = []
    for k in range(problem.T):
        order = None
        if problem.policy == "coord" and problem.coord_order is not None:
            order = np.ascontiguousarray(problem.coord_order[k], dtype=np.int64)
        steps.append((np.ascontiguousarray(problem.obs_idx[k], dtype=np.int64),
                      np.ascontiguousarray(problem.y[k], dtype=npdt),
                      np.ascontiguousarray(problem.noise_var[k], dtype=npdt), order))
    return steps


def run(handle, trans, inputs, smooth=True, reset=True):
    """Enqueue one full filter (+ smoother) pass; returns without synchronising."""
    if reset:
        handle.reset()
    for (A, Q), (idx, y, nv, order) in zip(trans, inputs):
        handle.predict(A, Q)
        if idx is None or len(idx) == 0:
            handle.update(None, None, None)
        else:
            handle.update(idx, y, nv, order)
        handle.truncate()
    if smooth:
        handle.smooth()


def collect(handle, T, which):
    means, vars_ = [], []
    for k in range(T + 1):
        m, v = handle.get(k, which)
        means.append(m.astype(np.float64))
        vars_.append(v.astype(np.float64))
    return means, vars_
