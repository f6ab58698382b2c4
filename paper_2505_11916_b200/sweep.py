"""Batched scenario sweeps: the evaluator's native entry point.

``evaluate_scenarios`` runs any list of (trace, config, rate scale)
scenarios in one persistent-kernel launch and returns per-scenario device
summaries (status, SLO attainment, P90/mean TTFT and TPOT, goodput, span,
flip count, decision-stream digest).  ``shard`` splits a sweep across
ranks for multi-GPU runs (scenarios are independent).
"""

from __future__ import annotations

import numpy as np

from ._buffers import OutputSpec
from ._compile import Scenario


def evaluate_scenarios(scenarios: list[Scenario], outputs: OutputSpec | None = None, evaluator=None):
    """Returns the HostBuffers of the launch (``.summaries`` is the
    arrow_summary_t array, one row per scenario, in input order)."""
    from .engine import execute

    _, hb = execute(scenarios, outputs or OutputSpec(), evaluator)
    return hb


def shard(n_items: int, rank: int, world: int) -> np.ndarray:
    """Static interleave: item i -> rank i % world (balances the rate/policy
    mix that drives per-scenario cost)."""
    return np.arange(rank, n_items, world, dtype=np.int64)
