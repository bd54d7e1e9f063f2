"""Seeded synthetic problem generators shared by the oracle tests, the GPU tests and bench.py.

This module holds none of the method's arithmetic: it only draws graphs, costs, capacities and
source/sink distributions (the BASELINE.json configs, SURVEY.md §8(d) table and the Q-readings of
SURVEY.md §8(c)).  Neither ``oracle/`` nor the CUDA library imports anything else from here.
"""
from .configs import Problem, gen, grid_problem, fig1_problem, CONFIG_NAMES  # noqa: F401
