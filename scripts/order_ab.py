"""A/B of work-queue orders for a multi-wave sweep (occupancy build):
does grouping scenarios that run the same code (policy, cluster size) onto
the GPU at the same time help the instruction caches?

    ARROW_C5_SAMPLE=16384 python scripts/order_ab.py
"""
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    from paper_2505_11916_b200 import engine
    from paper_2505_11916_b200._backend import CudaEvaluator
    from paper_2505_11916_b200._buffers import OutputSpec
    from paper_2505_11916_b200._compile import compile_batch, dispatch_order

    scen, _ = bench.workload("c5")
    ev = CudaEvaluator()
    cb = compile_batch(scen, engine.STALL_EVENT_LIMIT)
    base = dispatch_order(cb)          # shipped: (wide, policy, trace) groups, longest-first
    rank = np.empty(cb.n, dtype=np.int64)
    rank[base] = np.arange(cb.n)                       # longest-first position
    strat = cb.scenarios["strategy"].astype(np.int64)
    flips = cb.scenarios["enable_flips"].astype(np.int64)
    pol = strat * 2 + flips
    N = cb.scenarios["n_instances"].astype(np.int64)
    tr = np.asarray(cb.trace_index, dtype=np.int64)
    scale = cb.scenarios["arrival_scale"]
    theta = cb.scenarios["theta_d"] * 16 + cb.scenarios["theta_busy"] * 4 + cb.scenarios["breach_duration"]
    orders = {
        "shipped": base,
        "policy_trace_scale": np.lexsort((scale, tr, pol)).astype(np.int32),
        "policy_trace_N_scale": np.lexsort((scale, -N, tr, pol)).astype(np.int32),
        "policy_trace_longest_theta": np.lexsort((theta, rank, tr, pol)).astype(np.int32),
        "policy_trace_then_longest": np.lexsort((rank, tr, pol)).astype(np.int32),
    }
    res = {}
    for rep in range(2):
        for name, order in orders.items():
            db = ev.prepare(cb, OutputSpec(), order)
            ev.launch(db)
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            ev.launch(db)
            b.record()
            torch.cuda.synchronize()
            res.setdefault(name, []).append(a.elapsed_time(b))
    for name, v in res.items():
        print(f"{name:24s} " + " ".join(f"{x:8.1f} ms" for x in v))


if __name__ == "__main__":
    main()
