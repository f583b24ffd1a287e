"""FastPFP fp64 CPU oracle — TEST INFRASTRUCTURE (see oracle/fastpfp.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package. The product path never does.
"""
from .fastpfp import (  # noqa: F401
    FastPFP, Report, affinity, dykstra_project, edge_error, gradient, greedy_discretize, greedy_discretize_literal,
    objective, p1_affine, p2_nonneg, pd_project, project_loop, slack_embed, solve, sweep,
)
