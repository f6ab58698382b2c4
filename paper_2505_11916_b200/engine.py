"""Drop-in for pdsim.engine: ``run(trace, config) -> RunResult``.

The discrete-event loop itself (engine.py:122-316 of the reference) runs in
the CUDA evaluator; this module validates, compiles the scenario, launches
it and rebuilds the reference's RunResult.  ``STALL_EVENT_LIMIT`` is read at
call time, exactly like the reference (engine.py:119, 283), so tests that
monkeypatch it keep working.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

from . import _results
from ._buffers import OutputSpec
from ._compile import Scenario, compile_batch, dispatch_order
from .config import (  # noqa: F401  (re-exported like the reference module)
    CONFIG_KEYS as _CONFIG_KEYS,
    DEFAULTS as _DEFAULTS,
    RunConfig,
    config_from_values,
    default_run_config,
    load_run_config,
    parse_config_text,
)
from .core import PoolKind, RequestRecord, SLOConfig, TraceRequest  # noqa: F401
from .monitor import MonitorSnapshot

SimulationStallError = _results.SimulationStallError

# Abort if this many events pass without a token emitted or request finished.
STALL_EVENT_LIMIT = 500_000


@dataclass
class RunResult:
    records: list[RequestRecord]
    snapshots: list[MonitorSnapshot]
    decisions: list[dict]
    transitions: list[tuple[int, PoolKind, PoolKind]] = field(default_factory=list)


def scale_trace(trace: list[TraceRequest], s: float) -> list[TraceRequest]:
    """Arrival times multiplied by s (engine.py:94-98); the input is untouched."""
    if s <= 0:
        raise ValueError(f"scale factor must be positive, got {s}")
    return [replace(r, arrival=r.arrival * s) for r in trace]


FULL_OUTPUTS = OutputSpec(requests=True, decisions=True, snapshots=True, iterlog=True, diag=True)


def execute(scenarios: list[Scenario], spec: OutputSpec, evaluator=None, order=None):
    """Compile and run scenarios on the GPU, growing output buffers when a
    run reports an overflow.  Returns (CompiledBatch, HostBuffers)."""
    from ._backend import default_evaluator

    cb = compile_batch(scenarios, STALL_EVENT_LIMIT)
    # RunConfig.audit (engine.py:279-282): the per-step checking build
    audit = any(getattr(sc.config, "audit", False) for sc in scenarios)
    ev = evaluator or (default_evaluator(audit=True) if audit else default_evaluator())
    if order is None and cb.n > 1:
        order = dispatch_order(cb)
    while True:
        hb = ev.execute(cb, spec, order)
        ovf = hb.summaries["overflow"]
        if not (ovf != 0).any():
            return cb, hb
        grown = dict(spec.__dict__)
        for code, key in ((4, "decision_factor"), (5, "snapshot_factor"), (6, "iterlog_factor")):
            if (ovf == code).any():
                grown[key] *= 4
        if grown == spec.__dict__:
            return cb, hb
        spec = OutputSpec(**grown)


def result_from_buffers(cb, hb, s: int, config: RunConfig) -> RunResult:
    """The reference's RunResult (engine.py:86-91) for scenario s of a launch
    with FULL_OUTPUTS; raises the reference's exception for a failed run."""
    _results.raise_for_status(hb, s)
    entry = cb.table.entries[cb.trace_index[s]]
    decisions = _results.decision_dicts(hb, s, entry.ids)
    return RunResult(
        records=_results.records(hb, s, entry.arrival * float(cb.scenarios["arrival_scale"][s]), entry.ids,
                                 config.slo),
        snapshots=_results.snapshots(hb, s),
        decisions=decisions,
        transitions=_results.transitions(decisions),
    )


def run(trace: list[TraceRequest], config: RunConfig) -> RunResult:
    """Simulate a trace under a configuration; deterministic for fixed inputs."""
    cb, hb = execute([Scenario(trace, config, 1.0)], FULL_OUTPUTS)
    return result_from_buffers(cb, hb, 0, config)
