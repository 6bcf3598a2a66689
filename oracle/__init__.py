"""Plain fp64 CPU oracle for the BCFW semi-relaxed OT hot path (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package. The product path
(paper_2103_05857_b200) never imports it; the two share no code.
"""
from .oracle import *  # noqa: F401,F403
