"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no forces, kernels, lists):
only the input recipe of DESIGN.md §3 (positions, velocities, masses,
smoothing lengths, thermal energies and the parameter set, including the
grid-force polynomial that the method takes as an input).
"""
from .configs import make_config, make_params, CONFIGS  # noqa: F401
