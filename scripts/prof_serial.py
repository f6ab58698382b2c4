"""Serial-step cycle breakdown by event kind (needs a -DARROW_PROF build).

    ARROW_SIM_LIB=/tmp/libprof.so python scripts/prof_serial.py [c2|c5 [sample [trace digit]]]

c5: a seeded sample (default 4 096) of the C5 sweep through the occupancy
build; also prints the step counts (serial / parallel) and per-kind shares.
"""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2505_11916_b200 import engine, workloads as W
    from paper_2505_11916_b200._backend import CudaEvaluator, load_library
    from paper_2505_11916_b200._buffers import OutputSpec
    from paper_2505_11916_b200._compile import compile_batch, dispatch_order

    which = sys.argv[1] if len(sys.argv) > 1 else "c2"
    if which == "c5":
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
        ids = np.sort(np.random.default_rng(5).choice(98304, size=n, replace=False))
        if len(sys.argv) > 3:                       # restrict to one trace digit (0..3)
            ids = ids[ids % 4 == int(sys.argv[3])]
        scen = W.c5(ids)
    else:
        scen = W.c2(trace=W.c2_variant_trace(0))
    ev = CudaEvaluator()
    cb = compile_batch(scen, engine.STALL_EVENT_LIMIT)
    hb = ev.execute(cb, OutputSpec(), dispatch_order(cb))
    lib = load_library()
    out = np.zeros(len(scen) * 32, dtype=np.int64)
    rc = lib.arrow_sim_prof(out.ctypes.data_as(ctypes.c_void_p), len(scen))
    assert rc == 0, rc
    p = out.reshape(-1, 32)
    names = ["rr_iter", "rr_rank", "prefill_c", "arrival", "tick", "loud_iter", "migration", "rescan", "burst_sel",
             "burst_run", "round_sel", "round_run", "chains", "merge", "delays", "load_low", "sched_prefill",
             "sched_decode", "serial_tail", "iter_serial", "select_book"] + ["-"] * 11
    cyc = hb.summaries["cycles"]
    top = np.argsort(-cyc)[:6]
    for k in top:
        tot = cyc[k]
        parts = ", ".join(f"{names[q]} {100 * p[k, q] / tot:.1f}%" for q in range(21) if names[q] != "-")
        print(f"scenario {k}: {tot / 1e6:.1f}M cycles: {parts}")
    agg = p.sum(0) / cyc.sum()
    print("all:", ", ".join(f"{names[q]} {100 * agg[q]:.1f}%" for q in range(21) if names[q] != "-"))
    print("burst selections: attempted %d, past chain-safe test %d, ran %d" % tuple(p[:, 21:24].sum(0)))
    print("loud iterations: silent (no token) %d, PREFILL_COMPLETE-pushing %d" % (p[:, 25].sum(), p[:, 31].sum()))
    cnt = p[:, 24:32].sum(0)
    kinds = ["iter?", "-", "prefill_c", "arrival", "tick", "loud_iter", "migration", "-"]
    tot_cyc = cyc.sum()
    for q in (2, 3, 4, 5, 6):
        if cnt[q]:
            print(f"  {kinds[q]:10s} events {cnt[q]:12d}  cycles/event {p[:, q].sum() / cnt[q]:8.0f}")
    s = hb.summaries
    print("events %d serial steps %d parallel steps %d bursts+rounds; cycles/event %.0f" % (
        s["n_events"].sum(), s["n_serial_steps"].sum(), s["n_parallel_steps"].sum(), cyc.sum() / s["n_events"].sum()))


if __name__ == "__main__":
    main()
