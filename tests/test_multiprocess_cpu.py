"""Multi-rank sweep plumbing on CPU (gloo, world size 2): static interleaved
sharding of a scenario sweep and the final all-gather of per-scenario
summaries reproduce the single-process results exactly.  The CPU oracle
stands in for the per-rank GPU launch; the gather/assembly code is the one
bench.py uses with NCCL."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import harness as H
from paper_2505_11916_b200 import _abi
from paper_2505_11916_b200._buffers import OutputSpec
from paper_2505_11916_b200.sweep import (assemble_gathered, balanced_shards, gather_summaries, gather_summaries_into,
                                         shard, shard_bytes)

NAMES = ["small_arrow_2_2", "small_noflip", "rr_small", "fuzz_01", "fuzz_02", "fuzz_07", "fuzz_11"]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _items():
    idx = {m["name"]: m for m in H.golden_index()}
    return [(idx[n], H.golden_arrays(idx[n])) for n in NAMES]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    items = _items()
    limit = {m["stall_limit"] for m, _ in items}.pop()
    from paper_2505_11916_b200._compile import compile_batch, dispatch_estimate

    # bench.py's split: cost-balanced shards computed identically on every rank
    shards = balanced_shards(dispatch_estimate(compile_batch([H.golden_scenario(m, a) for m, a in items], limit))[0],
                             world)
    mine = shards[rank]
    cb = compile_batch([H.golden_scenario(*items[i]) for i in mine], limit)
    hb = H.run_oracle(cb, OutputSpec(), threads=1)
    full = gather_summaries(hb.summaries, len(items), rank, world, shards=shards)
    # the exact device-side path of bench.py (all_gather_into_tensor of
    # padded byte shards, then assembly in global order)
    local = torch.from_numpy(np.ascontiguousarray(hb.summaries).view(np.uint8).reshape(-1).copy())
    padded = torch.zeros(shard_bytes(len(items), world), dtype=torch.uint8)
    gathered = torch.empty(world * padded.numel(), dtype=torch.uint8)
    gather_summaries_into(local, padded, gathered)
    full2 = assemble_gathered(gathered.numpy(), len(items), world, shards)
    if rank == 0:
        q.put((full.tobytes(), full2.tobytes()))
    dist.destroy_process_group()


def test_sharded_sweep_gathers_to_single_process_result():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    data, data2 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gathered = np.frombuffer(data, dtype=_abi.SUMMARY_DTYPE)
    items = _items()
    from paper_2505_11916_b200._compile import compile_batch

    cb = compile_batch([H.golden_scenario(m, a) for m, a in items], items[0][0]["stall_limit"])
    ref = H.run_oracle(cb, OutputSpec(), threads=1).summaries
    assert gathered.tobytes() == ref.tobytes()
    assert data2 == ref.tobytes()            # bench.py's all_gather_into_tensor path
    for s, (m, a) in enumerate(items):
        assert H.bits(gathered[s]["attainment"]) == H.bits(m["summary"]["attainment"])


def test_shard_is_a_partition():
    rng = np.random.default_rng(0)
    for n in (1, 7, 96, 1000):
        for world in (1, 2, 4, 8):
            parts = np.concatenate([shard(n, r, world) for r in range(world)])
            assert sorted(parts.tolist()) == list(range(n))
            bal = balanced_shards(rng.random(n), world)
            assert sorted(np.concatenate(bal).tolist()) == list(range(n))
            assert max(len(b) for b in bal) - min(len(b) for b in bal) <= 1


def test_balanced_shards_mix_the_c5_radix():
    """C5 ids are trace-major: i % 8 would hand each of 8 ranks one trace;
    the cost-aware deal gives every rank every trace and policy."""
    from paper_2505_11916_b200 import engine
    from paper_2505_11916_b200 import workloads as W
    from paper_2505_11916_b200._compile import compile_batch, dispatch_estimate

    ids = np.arange(0, 98304, 7)
    cb = compile_batch(W.c5(ids), engine.STALL_EVENT_LIMIT)
    est = dispatch_estimate(cb)[0]
    for world in (2, 4, 8):
        shards = balanced_shards(est, world)
        loads = np.array([est[s].sum() for s in shards])
        assert loads.max() / loads.mean() < 1.01
        for s in shards:
            assert len(set(ids[s] % 4)) == 4                # every trace
            assert len(set(cb.scenarios["strategy"][s])) == 2 and len(set(cb.scenarios["enable_flips"][s])) == 2


def test_balanced_shards_ties_do_not_alias():
    """Scenarios the estimate cannot tell apart (equal est) carry hidden cost
    factors that follow the sweep's radix; the hashed tie-break and the
    back-and-forth deal spread them evenly (index order + round-robin put a
    period-2 factor entirely on the even ranks)."""
    n = 98304
    est = np.repeat(np.arange(n // 96, 0, -1, dtype=np.float64), 96)     # ties in runs of 96
    hidden = np.where(np.arange(n) % 2 == 0, 1.3, 1.0)                   # invisible to est
    for world in (2, 4, 8):
        shards = balanced_shards(est, world)
        loads = np.array([(est[s] * hidden[s]).sum() for s in shards])
        assert loads.max() / loads.mean() < 1.01, (world, loads / loads.mean())


def test_dispatch_order_runs_expensive_groups_first():
    """Groups (policy x trace) in decreasing mean estimate, longest-first
    inside each group; the cheapest group comes last."""
    from paper_2505_11916_b200 import engine
    from paper_2505_11916_b200 import workloads as W
    from paper_2505_11916_b200._compile import compile_batch, dispatch_estimate, dispatch_order

    ids = np.arange(0, 98304, 5)
    cb = compile_batch(W.c5(ids), engine.STALL_EVENT_LIMIT)
    est = dispatch_estimate(cb)[0]
    order = dispatch_order(cb)
    assert sorted(order.tolist()) == list(range(len(ids)))
    key = (ids % 4) * 8 + cb.scenarios["strategy"] * 2 + cb.scenarios["enable_flips"]
    k = key[order]
    starts = np.r_[0, np.nonzero(k[1:] != k[:-1])[0] + 1]
    assert len(starts) == len(np.unique(key))                            # each group contiguous
    means = [est[order[a:b]].mean() for a, b in zip(starts, np.r_[starts[1:], len(order)])]
    assert all(x >= y for x, y in zip(means, means[1:]))
    for a, b in zip(starts, np.r_[starts[1:], len(order)]):
        e = est[order[a:b]]
        assert (e[:-1] >= e[1:]).all()
