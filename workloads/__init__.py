"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the multi-scale method: it only draws
permeability fields K, source densities f and boundary-condition tables
according to the recipes in DESIGN.md §3.  Both sides of a
parity test consume exactly the same NumPy arrays produced here.
"""
from .configs import CONFIGS, Workload, make_workload, bc_table, random_problem  # noqa: F401
from .fields import gaussian_field  # noqa: F401
