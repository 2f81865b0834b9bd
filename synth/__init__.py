"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the method (no kernels, no SDE matrices, no
filtering).  It only builds the *inputs* of a workload: spatial grids (and their
R^3 embedding), the train/test split, time grids, observed values, noise
variances, hyperparameter values and policy inputs (coordinate orders).  Both
``oracle/`` and the CUDA path consume what it produces; neither imports the other.
"""
from .workloads import (  # noqa: F401
    Workload,
    grid_1d,
    sphere_grid,
    era5_test_mask,
    temperature_field,
    make_workload,
    WORKLOADS,
)
