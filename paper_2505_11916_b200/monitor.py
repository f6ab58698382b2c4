"""Monitor snapshot types (mirrors pdsim.monitor, monitor.py:19-41).

Snapshots are produced by the CUDA evaluator at every MONITOR_TICK
(before the scheduler's tick triggers, engine.py:250-253) when requested.
"""

from __future__ import annotations

from dataclasses import dataclass

from .core import PoolKind, SimTime


@dataclass(frozen=True)
class InstanceStats:
    instance_id: int
    pool: PoolKind
    running_tokens: int
    kv_used: int
    queue_len: int
    pred_delay: float
    avg_interval: float | None
    prefill_count: int
    decode_count: int


@dataclass(frozen=True)
class MonitorSnapshot:
    time: SimTime
    per_instance: tuple[InstanceStats, ...]

    def pool_counts(self) -> dict[PoolKind, int]:
        counts = dict.fromkeys(PoolKind, 0)
        for s in self.per_instance:
            counts[s.pool] += 1
        return counts
