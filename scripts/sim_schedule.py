"""Simulated multi-GPU schedule of the C5 sweep from measured per-scenario
cycles: bench's cost-balanced split (sweep.balanced_shards) and each rank's
work-queue order (_compile.dispatch_order), list-scheduled on 1 776 resident
warp slots per GPU.  Reports the makespan over a perfect split per N.

    python scripts/sim_schedule.py [gpurun_out/c5sum_r2u.npy]   (ARROW_BENCH_DUMP of a full C5 run)
"""
import heapq
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_11916_b200 import engine  # noqa: E402
from paper_2505_11916_b200 import workloads as W  # noqa: E402
from paper_2505_11916_b200 import _compile as C  # noqa: E402
from paper_2505_11916_b200.sweep import balanced_shards  # noqa: E402

SLOTS = 1776          # 148 SMs x 12 resident warps (occupancy build)
CLOCK = 1.965e9

cyc = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c5sum_r2u.npy")["cycles"].astype(float)
sc = W.c5()
t0 = time.time()
cb = C.compile_batch(sc, engine.STALL_EVENT_LIMIT)
t1 = time.time()
est = C.dispatch_estimate(cb)[0]
t2 = time.time()
C.dispatch_order(cb)
t3 = time.time()
print(f"compile {t1 - t0:.2f} s, estimate {t2 - t1:.3f} s, order {t3 - t2:.3f} s; "
      f"corr(estimate, cycles) {np.corrcoef(est, cyc)[0, 1]:.3f}")


def makespan(ids):
    sub = C.compile_batch([sc[i] for i in ids], engine.STALL_EVENT_LIMIT)
    h = [0.0] * SLOTS
    for x in cyc[ids][C.dispatch_order(sub)]:
        heapq.heappush(h, heapq.heappop(h) + x)
    return max(h)


for n in (1, 2, 4, 8):
    shards = balanced_shards(est, n) if n > 1 else [np.arange(len(sc))]
    worst = max(makespan(s) for s in shards)
    ideal = cyc.sum() / SLOTS / n
    loads = [cyc[s].sum() * n / cyc.sum() for s in shards]
    print(f"N={n}: makespan {worst / CLOCK:.3f} s, perfect split {ideal / CLOCK:.3f} s (+{100 * (worst / ideal - 1):.1f}%), "
          f"per-rank load {min(loads):.3f}-{max(loads):.3f} of the mean")
