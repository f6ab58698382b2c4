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
    """Static interleave: item i -> rank i % world."""
    return np.arange(rank, n_items, world, dtype=np.int64)


def balanced_shards(est: np.ndarray, world: int) -> list[np.ndarray]:
    """Cost-aware static split: scenarios sorted by estimated device time
    (``_compile.dispatch_estimate``) and dealt round-robin, so every rank gets
    the same mix of traces, rates, policies and cluster sizes.  A plain
    ``i % world`` interleave is not enough for mixed-radix sweeps: C5's
    scenario id is trace-major, so with 4 or 8 ranks each rank would get a
    single trace (C5 per-rank cycles max/mean: 1.72 interleaved, 1.02 dealt).
    Ties (scenarios the estimate cannot tell apart, e.g. two policies on the
    same trace and rate) are broken by a hash of the scenario index, and the
    deal runs back and forth (0..N-1, N-1..0): with index order and a plain
    round-robin, the sweep's mixed-radix structure aliases with the deal and
    puts the same hidden cost factor on the same ranks (C5 at 8 ranks:
    per-rank cost 0.83-1.20 of the mean).  Deterministic: every rank
    computes the same split."""
    est = np.asarray(est, dtype=np.float64)
    idx = np.arange(len(est), dtype=np.uint64)
    tie = (idx * np.uint64(0x9E3779B97F4A7C15)) >> np.uint64(32)     # Fibonacci hash
    order = np.lexsort((tie, -est))
    pos = np.arange(len(order))
    lap, r = pos // world, pos % world
    owner = np.empty(len(order), dtype=np.int64)
    owner[order] = np.where(lap % 2 == 0, r, world - 1 - r)
    return [np.nonzero(owner == q)[0] for q in range(world)]


def shard_bytes(n_total: int, world: int) -> int:
    """Bytes of one rank's padded summary shard (ceil(n / world) records)."""
    from ._abi import SUMMARY_DTYPE

    return -(-n_total // world) * SUMMARY_DTYPE.itemsize


def gather_summaries_into(local, padded, gathered) -> None:
    """Device-side all-gather of the per-scenario summaries (the sweep's only
    collective; NCCL over NVLink in bench.py, gloo in the CPU tests).

    local     uint8 tensor, this rank's summaries (n_local records)
    padded    uint8 tensor of shard_bytes(n_total, world) bytes (scratch)
    gathered  uint8 tensor of world * shard_bytes(...) bytes (output)
    """
    import torch.distributed as dist

    padded[: local.numel()].copy_(local)
    dist.all_gather_into_tensor(gathered, padded)


def assemble_gathered(gathered: np.ndarray, n_total: int, world: int, shards=None) -> np.ndarray:
    """Gathered shard bytes (rank-major) -> summaries in global scenario order
    (``shards``: each rank's global ids; default the static interleave)."""
    from ._abi import SUMMARY_DTYPE

    per = shard_bytes(n_total, world)
    raw = np.ascontiguousarray(gathered).view(np.uint8).reshape(world, per)
    full = np.zeros(n_total, dtype=SUMMARY_DTYPE)
    for r in range(world):
        ids = shard(n_total, r, world) if shards is None else shards[r]
        full[ids] = raw[r, : len(ids) * SUMMARY_DTYPE.itemsize].view(SUMMARY_DTYPE)
    return full


def gather_summaries(local: np.ndarray, n_total: int, rank: int, world: int, device=None,
                     shards=None) -> np.ndarray:
    """All-gather every rank's shard of per-scenario summaries (the sweep's
    only collective) and return them in global scenario order.  Shards are
    padded to equal size as collectives require."""
    import torch
    import torch.distributed as dist

    from ._abi import SUMMARY_DTYPE

    item = SUMMARY_DTYPE.itemsize
    per = -(-n_total // world)
    buf = torch.zeros(per * item, dtype=torch.uint8, device=device)
    raw = np.ascontiguousarray(local).view(np.uint8).reshape(-1)
    buf[: raw.size].copy_(torch.from_numpy(raw.copy()))
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    full = np.zeros(n_total, dtype=SUMMARY_DTYPE)
    for r in range(world):
        ids = shard(n_total, r, world) if shards is None else shards[r]
        data = outs[r].cpu().numpy()[: len(ids) * item]
        full[ids] = np.frombuffer(data.tobytes(), dtype=SUMMARY_DTYPE)
    return full
