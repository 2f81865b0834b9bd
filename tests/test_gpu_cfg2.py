"""End-to-end parity at BASELINE.json configs[1] (cfg2: D = 14,640 sphere grid, N = 5,580, 64
actions per step, rank cap 256) — the paper's policy-comparison size (Table C.1; App. C.3.1
P:2159-2176).  T = 6 so that the truncation is active at steps 5 and 6 (c = 320 > r = 256).

The oracle is the matrix-free O8 (oracle/mfree.py, pinned to the dense O4/O5 in
tests/test_oracle_mfree.py) with its kernel matrices cached.
  * random / coordinate actions (fixed, data-independent): fp64 within 1e-9 (north_star);
  * CG actions (residual-dependent Krylov trajectory, R20): fp64 judged against the oracle's own
    sensitivity to a 1-ulp relative perturbation of y;
  * fp32: means within 1e-4 and variances within the downdate-cancellation bound of R20 for the
    fixed-action policies; CG in fp32 is reported (R20: "reported, not gated") and must keep every
    variance positive.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import mfree  # noqa: E402
from paper_2405_08971_b200 import CAKF_FILTER, CAKF_SMOOTH, runner  # noqa: E402
from synth import make_workload  # noqa: E402

EPS32 = float(np.finfo(np.float32).eps)
_ORACLE = {}


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def workload(policy):
    return make_workload("cfg2", policy=policy, T=6)


def oracle(policy, dtype, perturb=0.0):
    key = (policy, dtype, perturb)
    if key not in _ORACLE:
        wl = workload(policy)
        _ORACLE[key] = mfree.run_mf(wl, dtype_round=np.float32 if dtype == "f32" else None, cache=True,
                                    perturb_y=perturb)
    return _ORACLE[key]


def device(policy, dtype):
    wl = workload(policy)
    trans, _ = runner.transitions(wl)
    h = runner.make_handle(wl, dtype)
    runner.run(h, trans, runner.stage_inputs(wl, dtype), smooth=True)
    h.sync()
    out = {}
    out["fm"], out["fv"] = runner.collect(h, wl.T, CAKF_FILTER)
    out["sm"], out["sv"] = runner.collect(h, wl.T, CAKF_SMOOTH)
    out["stats"] = [h.get_stats(k) for k in range(wl.T + 1)]
    h.destroy()
    return wl, out


def _mrel(x, y):
    """R20: ||dm||_inf / ||m||_inf; a zero reference mean (the prior at k = 0) must be matched exactly."""
    den = float(np.max(np.abs(y)))
    num = float(np.max(np.abs(x - y)))
    return num / den if den > 0 else (0.0 if num == 0 else np.inf)


def rel_errs(a, b):
    m = max(_mrel(x, y) for key in ("fm", "sm") for x, y in zip(a[key], b[key]))
    v = max(float(np.max(np.abs(x - y) / np.abs(y))) for key in ("fv", "sv") for x, y in zip(a[key], b[key]))
    return m, v


def heldout_rmse(wl, means):
    """RMSE of the filter / smoother mean of f_0 on the held-out test subgrid vs the noise-free field."""
    from synth.workloads import temperature_field
    X = wl.coords[wl.test_idx]
    lat, lon = np.arcsin(np.clip(X[:, 2], -1, 1)), np.arctan2(X[:, 1], X[:, 0])
    errs = [means[k][wl.test_idx] - temperature_field(wl.times[k - 1], lat, lon) for k in range(1, wl.T + 1)]
    return float(np.sqrt(np.mean(np.concatenate(errs) ** 2)))


def check_ranks(wl, out):
    cols = 0
    for k in range(1, wl.T + 1):
        st = out["stats"][k]
        assert st["iters"] == wl.max_iter
        assert st["rank_in"] == cols and st["cols"] == cols + wl.max_iter
        cols = min(wl.max_rank, cols + wl.max_iter)
        assert st["rank_out"] == cols
    assert out["stats"][wl.T]["rank_out"] == 256 and out["stats"][5]["cols"] == 320   # truncation active


def positive(out):
    for key in ("fv", "sv"):
        for k, v in enumerate(out[key]):
            assert np.min(v) > 0, (key, k, float(np.min(v)))


@pytest.mark.parametrize("policy", ["random", "coord"])
def test_cfg2_fixed_actions_fp64(policy):
    wl, out = device(policy, "f64")
    check_ranks(wl, out)
    positive(out)
    m, v = rel_errs(out, oracle(policy, "f64"))
    print(f"cfg2 {policy} fp64: mean {m:.3g} var {v:.3g}")
    assert m < 1e-9 and v < 1e-9


@pytest.mark.parametrize("policy", ["random", "coord"])
def test_cfg2_fixed_actions_fp32(policy):
    wl, out = device(policy, "f32")
    check_ranks(wl, out)
    positive(out)
    ref = oracle(policy, "f32")
    m, v = rel_errs(out, ref)
    print(f"cfg2 {policy} fp32: mean {m:.3g} var {v:.3g}")
    assert m < 1e-4
    sdd = wl.sigma ** 2 * 3.0 / wl.ell_t ** 2   # Sigma_inf[1,1]; Sigma^t_dd <= max(sigma^2, this) for all k
    bound_abs = 2048 * EPS32 * max(wl.sigma ** 2, sdd)
    for key in ("fv", "sv"):
        for x, y in zip(out[key], ref[key]):
            assert np.all(np.abs(x - y) <= 1e-4 * y + bound_abs)


@pytest.mark.parametrize("iters,rank", [(2, 4), (6, 16)])
def test_cfg2_cg_short_fp64(iters, rank):
    """CG actions while the Krylov trajectory is still well-conditioned, rank cap below the column
    count so the truncation is active from step 3.  The oracle's own sensitivity to a 1-ulp relative
    perturbation of y grows fast with the iterations at cfg2 (1.5e-11 at 2, 1e-9 at 4,
    2e-8 at 6 iterations per step over 6 steps), so: 2 iterations -> fp64 within 1e-9 (north_star);
    6 iterations -> within 16x the oracle's measured 1-ulp sensitivity (a different but equally valid
    rounding in each of the 36 Krylov steps)."""
    wl = make_workload("cfg2", policy="cg", T=6, max_iter=iters, max_rank=rank)
    trans, _ = runner.transitions(wl)
    h = runner.make_handle(wl, "f64")
    runner.run(h, trans, runner.stage_inputs(wl, "f64"), smooth=True)
    out = {}
    out["fm"], out["fv"] = runner.collect(h, wl.T, CAKF_FILTER)
    out["sm"], out["sv"] = runner.collect(h, wl.T, CAKF_SMOOTH)
    ranks = [h.get_stats(k)["rank_out"] for k in range(1, wl.T + 1)]
    h.destroy()
    assert ranks == [min(rank, iters * k) for k in range(1, wl.T + 1)]
    positive(out)
    ref = mfree.run_mf(wl, cache=True)
    m, v = rel_errs(out, ref)
    sm_, sv_ = rel_errs(mfree.run_mf(wl, cache=True, perturb_y=2.0 ** -52), ref)
    print(f"cfg2 cg ({iters} iterations) fp64: mean {m:.3g} var {v:.3g}; oracle 1-ulp sensitivity {sm_:.3g} {sv_:.3g}")
    if iters <= 2:
        assert m < 1e-9 and v < 1e-9
    else:
        assert m <= 16 * sm_ and v <= 16 * sv_


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_cfg2_cg_64_reported_against_oracle_sensitivity(dtype):
    """64 CG iterations per step (the bench's policy): the oracle itself moves O(1) under a 1-ulp
    relative perturbation of y (R20: the Krylov trajectory amplifies rounding ~8x per
    iteration), so element-wise parity is undefined here.  Reported: device-vs-oracle error next to
    the oracle's own 1-ulp sensitivity.  Gated: every variance positive, and the held-out RMSE of the
    device's means (a property every valid trajectory shares) within the oracle-vs-perturbed-oracle
    spread of the oracle's RMSE (x3, + 5 %)."""
    wl, out = device("cg", dtype)
    check_ranks(wl, out)
    positive(out)
    ref = oracle("cg", dtype)
    pert = oracle("cg", dtype, perturb=2.0 ** -52)
    m, v = rel_errs(out, ref)
    sm_, sv_ = rel_errs(pert, ref)
    print(f"cfg2 cg {dtype}: device-vs-oracle mean {m:.3g} var {v:.3g}; oracle 1-ulp sensitivity "
          f"mean {sm_:.3g} var {sv_:.3g}")
    for key in ("fm", "sm"):
        r_dev, r_or, r_pt = heldout_rmse(wl, out[key]), heldout_rmse(wl, ref[key]), heldout_rmse(wl, pert[key])
        print(f"  {key} held-out RMSE: device {r_dev:.4f} oracle {r_or:.4f} perturbed oracle {r_pt:.4f}")
        assert abs(r_dev - r_or) <= 3 * abs(r_pt - r_or) + 0.05 * r_or
