"""Seeded synthetic workload generators shared by the oracle and the CUDA harness.

This package holds ONLY input generation: program DAGs, call lengths, arrival
steps and token contexts.  It contains none of the scheduling method's
arithmetic (no priorities, queues, cutoffs, routing or swap accounting), so
that `oracle/` and `paper_2502_13965_b200/` can both consume the same traces
without sharing any method code (task rule ③).
"""
from .gen import (  # noqa: F401
    Trace, fig2, atlas_dag_fixture, random_tiny, chatbot, react, mcts_mapreduce,
    mixed, burst_mcts_mapreduce, burst_mixed, churn, concat, lognormal_clipped, dag_trace, BASE_SEED,
    CONFIG_INDEX,
)
