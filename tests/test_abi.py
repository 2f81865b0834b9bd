"""C-ABI checks that need no GPU: the library loads, exports every declared symbol,
its host-only entry points behave, and errors are reported (not silently ignored)."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import model
from paper_2405_08971_b200 import binding

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2405_08971_b200 import build
    build.build()
    return binding.load()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "cakf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(\w+)\s*\(", src, flags=re.M)))


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(binding.EXPORTS)
    assert lib.cakf_version() == 1


@pytest.mark.parametrize("nu", [0.5, 1.5, 2.5])
def test_matern_transition_matches_oracle(lib, nu):
    """Closed forms in the library vs expm + Lyapunov in the oracle (independent)."""
    for ell, sigma, dt in [(0.5, 1.0, 0.1), (3.0, 10.0, 1.0), (0.7, 2.0, 0.0), (1.3, 0.5, 2.5)]:
        A, Q, S = binding.matern_transition(nu, ell, sigma, dt)
        Ao, Qo, So = model.temporal_transition(nu, ell, sigma, dt)
        scale = max(1.0, np.abs(So).max())
        assert np.allclose(A, Ao, rtol=1e-10, atol=1e-12)
        assert np.allclose(S, So, rtol=1e-10, atol=1e-10 * scale)
        assert np.allclose(Q, Qo, rtol=1e-9, atol=1e-9 * scale)


def test_errors_are_reported(lib):
    h = ctypes.c_void_p()
    assert lib.cakf_create(None, ctypes.byref(h)) == -1
    assert b"NULL" in lib.cakf_last_error()
    cfg = binding.cakf_config(dtype=0, d_time=2, n_space=4, space_dim=5)
    assert lib.cakf_create(ctypes.byref(cfg), ctypes.byref(h)) == -1
    assert lib.cakf_predict(None, None, None, None) == -1
    assert lib.cakf_matern_transition(4, 1.0, 1.0, 0.1, None, None, None) == -3


def test_create_without_gpu_fails_loudly(lib):
    """No CPU fallback: on a machine without a CUDA device cakf_create must fail."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(binding.CakfError):
        binding.Cakf(np.zeros((4, 1)), 1.0, np.eye(2), dtype="f32", max_steps=2)
