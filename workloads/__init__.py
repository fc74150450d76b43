"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds *no* arithmetic of the ParaDiag method: only problem parameter
tables (BASELINE.json ``configs``) and the counter-based generator that fills the
initial data u0.  Both the oracle (``oracle/``) and the CUDA path
(``paper_2304_14021_b200``) receive their inputs from here, so the two sides see
identical bits.
"""
from .configs import Problem, CONFIGS, config, twin  # noqa: F401
from .rng import splitmix64, uniform, make_u0, grid_coords  # noqa: F401
