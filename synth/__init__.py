"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the paper's method (no power-flow
equations, no derivatives, no reductions): it only draws topologies,
π-model line admittances (MATPOWER convention, the paper omits them —
SURVEY §2.1 A2), operating points and IPM-like multipliers, with the
shapes of the paper's Table 1 instances.
"""
from .case9 import case9
from .grid import make_grid, make_scenario, counts, TABLE1

__all__ = ["case9", "make_grid", "make_scenario", "counts", "TABLE1"]
