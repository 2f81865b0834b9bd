"""B200-native computation-aware Kalman filter / RTS smoother (CAKF/CAKS, arXiv 2405.08971).

The product is ``libcakf.so`` (C-ABI declared in ``include/cakf.h``, hand-written
sm_100a CUDA kernels); ``binding`` is its thin ctypes wrapper and ``runner`` the
host-side call sequence (predict -> update -> truncate per step, then smooth).
"""
from .binding import (  # noqa: F401
    CAKF_FILTER,
    CAKF_PRED,
    CAKF_SMOOTH,
    Cakf,
    CakfError,
    gram_matmul,
    load,
    matern_transition,
)
