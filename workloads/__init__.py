"""Seeded synthetic inputs for CrossPipe (arXiv 2507.00217) -- shared by the oracle
side (tests) and the product side (bench/tests).

This module holds NO arithmetic of the method: no timeline recurrence, no link
model, no greedy rule, no memory accounting of timelines.  It only builds problem
instances (integer ticks / memory units), sweep grids, and random *valid* plans
(a combinatorial token game, see gen.cu), plus pure format conversions
(2-bit packing).  Recipes follow SURVEY.md §8(d); DESIGN.md §Inputs restates them.
"""
from .core import (  # noqa: F401
    F, B, D, W, MAXP, InstanceBatch, Grid, splitmix64, pack_plans, unpack_plans,
    cross_dc_boundaries,
)
from . import configs  # noqa: F401
