"""Whole-sweep digests from the REAL reference (TEST INFRASTRUCTURE; build
container only).

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden_digest.py c3|c4|c5[:N] [workers]

Runs every scenario of the BASELINE C3 (1 920) or C4 (1 080) sweep -- or a
seeded sample of N C5 ids -- through the real ``pdsim.run`` on a process
pool and stores, per scenario: the status (ok / stalled at time t), every
RunSummary field, the number of decisions and flips, and the FNV-1a digest of
the decision stream computed exactly like the kernel's (oracle/pdsim_oracle.c:
pdsim_oracle_decision_hash over the encoded decision records), in
tests/golden/digest_<set>.npz.  tests/test_gpu_sweeps.py runs the same ids
through the CUDA evaluator (paper_2505_11916_b200/workloads.py) and requires
every field to match bit for bit.
"""

from __future__ import annotations

import ctypes
import multiprocessing as mp
import sys
import time
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(ROOT))

SUMMARY = ("attainment", "p90_ttft", "p90_tpot", "mean_ttft", "mean_tpot", "goodput", "span_s")
_cache: dict = {}


def _traces(which):
    import pdsim
    import scenarios as S

    if which not in _cache:
        mk = pdsim.TraceRequest
        if which == "c3":
            _cache[which] = [S.code_like(mk), S.conversation_like(mk)]
        elif which == "c4":
            _cache[which] = S.c4_trace(mk)
        else:
            _cache[which] = [S.bursty(mk), S.code_like(mk), S.conversation_like(mk), S.ramp(mk)]
    return _cache[which]


def run_one(args):
    which, sid = args
    import pdsim
    import pdsim.engine as E
    import scenarios as S

    from gen_golden import encode_decisions
    from paper_2505_11916_b200 import _abi

    mk = pdsim.TraceRequest
    if which == "c3":
        trace, v, scale = S.c3_scenario(mk, sid, _traces("c3"))
    elif which == "c4":
        trace, v, scale = S.c4_scenario(mk, sid, _traces("c4"))
    else:
        trace, v, scale = S.c5_scenario(mk, sid, _traces("c5"))
    t0 = time.perf_counter()
    out = dict(id=sid, status=0, stall_time=np.nan, n_decisions=0, n_flips=0, decision_hash=0)
    try:
        res = pdsim.run(pdsim.scale_trace(trace, scale), pdsim.config_from_values(v))
        s = pdsim.compute_metrics(res.records, pdsim.config_from_values(v).slo).to_dict()
        for k in SUMMARY:
            out[k] = s[k]
        dec = encode_decisions(res.decisions, {r.id: i for i, r in enumerate(trace)})
        arr = np.zeros(len(dec), dtype=_abi.DECISION_DTYPE)
        for f in dec.dtype.names:
            arr[f] = dec[f]
        lib = ctypes.CDLL(str(HERE / "build" / "libpdsim_oracle.so"))
        lib.pdsim_oracle_decision_hash.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        lib.pdsim_oracle_decision_hash.restype = ctypes.c_uint64
        out["decision_hash"] = int(lib.pdsim_oracle_decision_hash(arr.ctypes.data, len(arr)))
        out["n_decisions"] = len(arr)
        out["n_flips"] = len(res.transitions)
    except E.SimulationStallError as exc:
        out["status"] = 1
        out["stall_time"] = float(str(exc).split("t=", 1)[1].split(":", 1)[0])
        for k in SUMMARY:
            out[k] = np.nan
    out["wall_s"] = time.perf_counter() - t0
    return out


def main() -> None:
    which = sys.argv[1]
    workers = int(sys.argv[2]) if len(sys.argv) > 2 else 7
    if which == "c3":
        ids = np.arange(1920)
    elif which == "c4":
        ids = np.arange(1080)
    elif which.startswith("c5"):
        n = int(which.split(":")[1]) if ":" in which else 256
        ids = np.sort(np.random.default_rng(5005).choice(98304, size=n, replace=False))
        which = "c5"
    else:
        raise SystemExit(which)
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(workers) as pool:
        rows = []
        for k, r in enumerate(pool.imap_unordered(run_one, [(which, int(i)) for i in ids], chunksize=1)):
            rows.append(r)
            if k % 100 == 0:
                print(f"{k}/{len(ids)} {time.perf_counter() - t0:.0f}s", flush=True)
    rows.sort(key=lambda r: r["id"])
    arrays = {k: np.array([r[k] for r in rows]) for k in rows[0]}
    arrays["decision_hash"] = np.array([r["decision_hash"] for r in rows], dtype=np.uint64)
    tag = "c5" if which == "c5" else which
    np.savez_compressed(ROOT / "tests" / "golden" / f"digest_{tag}.npz", **arrays)
    print(f"{len(rows)} scenarios, {int((arrays['status'] == 1).sum())} stalls, {time.perf_counter() - t0:.0f}s")


if __name__ == "__main__":
    main()
