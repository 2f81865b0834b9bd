"""Full-size parity on sampled outputs: the fused kernel operators at BASELINE.json's
cfg3 shapes (N_X = 115,680 points, N = 87,120 training points), checked row by row against
the oracle's chunked kernel rows.  `test_k1_bench_launch_path_cfg3` runs K1 through the handle's
own inner-loop launch path (cakf_debug_matvec: kd order, exact-zero culling lists, dynamic unit
scheduler, partial slots) — the configuration the bench times; the cakf_gram_matmul tests run
the standalone operator (no culling lists)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import mfree  # noqa: E402
from paper_2405_08971_b200 import binding  # noqa: E402
from synth import make_workload  # noqa: E402


@pytest.fixture(scope="module")
def cfg3():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return make_workload("cfg3", T=1)


def _rel_err(got, ref, X, xr, xc, nu, ell):
    scale = np.abs(mfree.gram_apply(xr, xc, np.abs(X), nu, ell, chunk=256))
    return float(np.max(np.abs(got - ref) / np.maximum(scale, 1e-300)))


@pytest.mark.parametrize("ncols", [1, 65, 1026])
def test_gram_operator_cfg3_sampled_rows(cfg3, ncols):
    """K1 (ncols = 1, rows x train) and K2 (post-loop 65 / smoother 1026 columns, rows x all):
    the first 256 and last 128 rows (ragged tail) of the full-size product vs the oracle."""
    wl = cfg3
    rng = np.random.default_rng(ncols)
    X_all = wl.coords
    cols = X_all[wl.obs_idx[0]] if ncols == 1 else X_all
    B = rng.standard_normal((len(cols), ncols))
    dev = "cuda"
    rows = np.concatenate([np.arange(256), np.arange(len(X_all) - 128, len(X_all))])
    xr = torch.tensor(X_all[rows].astype(np.float32), device=dev)
    xc = torch.tensor(cols.astype(np.float32), device=dev)
    Bt = torch.tensor(B.astype(np.float32), device=dev)
    Y = binding.gram_matmul(xr, xc, Bt[:, 0] if ncols == 1 else Bt, wl.nu_x, wl.ell_x)
    Y = Y.double().cpu().numpy().reshape(len(rows), -1)
    xr64 = X_all[rows].astype(np.float32).astype(np.float64)
    xc64 = cols.astype(np.float32).astype(np.float64)
    B64 = B.astype(np.float32).astype(np.float64)
    ref = mfree.gram_apply(xr64, xc64, B64, wl.nu_x, wl.ell_x, chunk=64)
    err = _rel_err(Y, ref, B64, xr64, xc64, wl.nu_x, wl.ell_x)
    print("cfg3 sampled rows, ncols", ncols, "max rel err", err)
    assert err < 2e-5


def test_symmetric_k1_cfg3(cfg3):
    """The inner-loop matvec K_TT s (symmetric tile-pair kernel, N = 87,120) at full size:
    sampled rows vs the oracle, and all rows vs the dense-kernel path."""
    wl = cfg3
    rng = np.random.default_rng(7)
    Xt = wl.coords[wl.obs_idx[0]]
    s = rng.standard_normal(len(Xt))
    xt = torch.tensor(Xt.astype(np.float32), device="cuda")
    st = torch.tensor(s.astype(np.float32), device="cuda")
    y = binding.gram_matmul(xt, xt, st, wl.nu_x, wl.ell_x).double().cpu().numpy()      # xr is xc: symmetric
    y_dense = binding.gram_matmul(xt, xt.clone(), st, wl.nu_x, wl.ell_x).double().cpu().numpy()
    rows = np.concatenate([np.arange(200), np.arange(len(Xt) - 77, len(Xt))])
    X64 = Xt.astype(np.float32).astype(np.float64)
    s64 = s.astype(np.float32).astype(np.float64)
    ref = mfree.gram_apply(X64[rows], X64, s64, wl.nu_x, wl.ell_x, chunk=64)
    scale = mfree.gram_apply(X64[rows], X64, np.abs(s64), wl.nu_x, wl.ell_x, chunk=64)
    err = float(np.max(np.abs(y[rows] - ref) / scale))
    err_all = float(np.max(np.abs(y - y_dense) / np.maximum(np.abs(y_dense), 1e-30)))
    print("symmetric K1 cfg3: sampled rel err", err, "vs dense kernel", err_all)
    assert err < 1e-6
    assert np.max(np.abs(y - y_dense)) < 1e-5 * np.max(np.abs(y_dense))


def test_k1_bench_launch_path_cfg3(cfg3):
    """K1 at N = 87,120 exactly as cakf_update launches it in the bench (fp32, culling on, dynamic
    scheduler, kd-ordered observations): sampled rows vs the oracle, plus every row vs the same
    handle with culling off (exact-zero culling changes no bit: DESIGN §6)."""
    from paper_2405_08971_b200 import runner
    wl = cfg3
    rng = np.random.default_rng(11)
    idx = wl.obs_idx[0]
    s = rng.standard_normal(len(idx))
    outs = {}
    for cull in (True, False):
        h = runner.make_handle(wl, "f32", cull_zero=cull)
        outs[cull] = h.debug_matvec(idx, s.astype(np.float32)).astype(np.float64)
        again = h.debug_matvec(idx, s.astype(np.float32)).astype(np.float64)   # cached order, same bits
        assert np.array_equal(again, outs[cull])
        # the multi-GPU split of K1 (8 and 3 ranks' unit shares, balanced by active tile pairs with culling,
        # by unit index without) covers every unit exactly once: the same bits as one launch
        for shares in (8, 3):
            assert np.array_equal(h.debug_matvec(idx, s.astype(np.float32), shares=shares).astype(np.float64),
                                  outs[cull])
        h.destroy()
    assert np.array_equal(outs[True], outs[False])
    y = outs[True]
    # the handle stores the coordinates prescaled by sqrt(2 nu)/ell and rounded once to fp32; the oracle
    # takes exactly those inputs (in fp64) with the matching lengthscale sqrt(2 nu), so the comparison
    # isolates the kernel's arithmetic from the input rounding (which near the poles alone moves the
    # small distances by ~1e-4 relative)
    sc = np.sqrt(2 * wl.nu_x) / wl.ell_x
    Xt = (wl.coords[idx] * sc).astype(np.float32).astype(np.float64)
    s64 = s.astype(np.float32).astype(np.float64)
    ell_s = np.sqrt(2 * wl.nu_x)
    rows = np.concatenate([np.arange(200), np.arange(len(idx) - 77, len(idx)), rng.choice(len(idx), 200, replace=False)])
    ref = mfree.gram_apply(Xt[rows], Xt, s64, wl.nu_x, ell_s, chunk=64)
    scale = mfree.gram_apply(Xt[rows], Xt, np.abs(s64), wl.nu_x, ell_s, chunk=64)
    err = float(np.max(np.abs(y[rows] - ref) / scale))
    print("K1 bench launch path cfg3: sampled rel err", err)
    assert err < 1e-6


def test_exact_zero_culling_is_bit_identical_cfg3():
    """Exact-zero culling skips only kernel tiles whose every fp32 value is exactly 0,
    so the filter and smoother outputs with culling on and off must be bit-identical, while a
    real share of the K1 / K2 tiles is skipped at cfg3's lengthscale."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2405_08971_b200 import CAKF_FILTER, CAKF_SMOOTH, runner
    wl = make_workload("cfg3", T=3, max_iter=24, max_rank=48)
    trans = runner.transitions(wl)[0]
    inputs = runner.stage_inputs(wl, "f32")
    outs, fracs = [], []
    for cull in (False, True):
        h = runner.make_handle(wl, "f32", cull_zero=cull)
        runner.run(h, trans, inputs)
        h.sync()
        outs.append([runner.collect(h, wl.T, w) for w in (CAKF_FILTER, CAKF_SMOOTH)])
        fracs.append(h.cull_stats())
        h.destroy()
    for a, b in zip(outs[0], outs[1]):
        for ka, kb in zip(a[0] + a[1], b[0] + b[1]):
            assert np.array_equal(ka, kb)
    assert fracs[0] == {"k1_matvec": 1.0, "k2_post": 1.0, "k2_smooth": 1.0}
    print("cull fractions", fracs[1])
    assert all(0.0 < f < 0.9 for f in fracs[1].values())


def test_cfg4_maximum_size():
    """The largest configuration (BASELINE cfg4: N_X = 501,000, D = 1,002,000, N = 376,500,
    r = 1024) on one GPU: the symmetric K1 at N = 376,500 on sampled rows vs the oracle, and a
    3-step filter + smoother pass whose outputs are finite and within [0, prior] variance."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2405_08971_b200 import CAKF_FILTER, CAKF_SMOOTH, runner
    wl = make_workload("cfg4", T=3)
    Xt = wl.coords[wl.obs_idx[0]]
    rng = np.random.default_rng(4)
    s = rng.standard_normal(len(Xt))
    xt = torch.tensor(Xt.astype(np.float32), device="cuda")
    y = binding.gram_matmul(xt, xt, torch.tensor(s.astype(np.float32), device="cuda"), wl.nu_x,
                            wl.ell_x).double().cpu().numpy()
    rows = np.concatenate([np.arange(128), np.arange(len(Xt) - 61, len(Xt))])
    X64 = Xt.astype(np.float32).astype(np.float64)
    s64 = s.astype(np.float32).astype(np.float64)
    ref = mfree.gram_apply(X64[rows], X64, s64, wl.nu_x, wl.ell_x, chunk=32)
    scale = mfree.gram_apply(X64[rows], X64, np.abs(s64), wl.nu_x, wl.ell_x, chunk=32)
    assert float(np.max(np.abs(y[rows] - ref) / scale)) < 1e-6
    del xt
    trans, Sinf = runner.transitions(wl)
    h = runner.make_handle(wl, "f32")
    runner.run(h, trans, runner.stage_inputs(wl, "f32"))
    h.sync()
    prior = np.repeat(np.diag(Sinf), wl.n_space)
    for k in range(wl.T + 1):
        for which in (CAKF_FILTER, CAKF_SMOOTH):
            m, v = h.get(k, which)
            assert np.all(np.isfinite(m)) and np.all(np.isfinite(v))
            assert np.all(v <= prior * (1 + 1e-5)) and np.all(v > 0), (k, which, float(np.min(v)))
    assert [h.get_stats(k)["rank_out"] for k in range(1, wl.T + 1)] == [64, 128, 192]
    assert 0.0 < h.cull_stats()["k1_matvec"] < 0.2
    h.destroy()
