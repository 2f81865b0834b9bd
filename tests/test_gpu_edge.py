"""Edge cases of the device path vs the oracle (fp64, 1e-9): single observations, more iterations
than observations, one time step, observation sets that change size and membership every step
(per-update device sort + kd order), a 3-point grid, and all points observed."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import make_workload  # noqa: E402
from test_gpu_parity import compare  # noqa: E402


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _reobserve(wl, sets, seed=0):
    rng = np.random.default_rng(seed)
    for k, idx in enumerate(sets):
        idx = np.asarray(idx, dtype=np.int64)
        wl.obs_idx[k] = idx
        wl.y[k] = rng.standard_normal(len(idx))
        wl.noise_var[k] = np.full(len(idx), wl.lam ** 2) * (1.0 + 0.5 * rng.random(len(idx)))
    return wl


def test_single_observation_per_step():
    wl = make_workload("line8", T=5, policy="cg", max_iter=3, max_rank=3)
    _reobserve(wl, [[k % 8] for k in range(wl.T)])
    compare(wl, "f64", 1e-9, 1e-9)


def test_more_iterations_than_observations():
    wl = make_workload("line8", T=4, policy="cg", max_iter=20, max_rank=-1)
    compare(wl, "f64", 1e-9, 1e-9)


def test_one_time_step():
    wl = make_workload("sphere48", T=1, policy="cg", max_iter=8, max_rank=4)
    compare(wl, "f64", 1e-9, 1e-9)


@pytest.mark.parametrize("policy", ["cg", "random"])
def test_changing_observation_sets(policy):
    wl = make_workload("sphere48", T=5, policy=policy, max_iter=12, max_rank=20)
    n = wl.n_space
    rng = np.random.default_rng(3)
    sets = [np.sort(rng.choice(n, size=m, replace=False)) for m in (n, 37, 1, 0, n // 2)]
    _reobserve(wl, sets)
    compare(wl, "f64", 1e-9, 1e-9)


def test_three_point_grid():
    wl = make_workload("line8", n=3, T=4, policy="cg", max_iter=2, max_rank=2, test_every=0)
    compare(wl, "f64", 1e-9, 1e-9)


def test_observation_cache_device_and_host_pointers():
    """Same-size sets that alternate membership (A, A, B, B, A, A): the observation-order cache is decided on
    the device for device-pointer obs_idx (no host round trip) and on the host for host arrays.  Both paths
    must match the oracle and each other bit for bit (the order is a pure function of obs_idx)."""
    wl = make_workload("sphere48", T=6, policy="cg", max_iter=10, max_rank=16)
    n = wl.n_space
    rng = np.random.default_rng(11)
    A = np.sort(rng.choice(n, size=n // 3, replace=False))
    B = np.sort(rng.choice(n, size=n // 3, replace=False))
    _reobserve(wl, [A, A, B, B, A, A[::-1].copy()])
    _, errs = compare(wl, "f64", 1e-9, 1e-9, on_device=True)
    from test_gpu_parity import run_device
    dev = run_device(wl, "f64", on_device=True)
    host = run_device(wl, "f64", on_device=False)
    for a, b in zip(dev[1:5], host[1:5]):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
