"""Seeded synthetic input generators shared by tests, bench.py and smoke().

This module holds NONE of the method's arithmetic (no LMO, gap, step size or
update). It only builds problem inputs — colours, marginals, costs — with the
shapes and distributions of BASELINE.json's configs (DESIGN.md §4 recipe).
Both the oracle (oracle/) and the CUDA path receive identical arrays from it.
"""
from .gen import *  # noqa: F401,F403
