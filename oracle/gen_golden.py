"""Generate tests/golden/ from the REAL reference (TEST INFRASTRUCTURE).

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden.py

Imports pdsim from /root/reference/pkg/src (read-only, only present in the
build container), runs every scenario of oracle/scenarios.py through
``pdsim.run`` and stores inputs + outputs as small npz/json fixtures.  The
GPU box never needs /root/reference: tests read only the fixtures.

Also records known-answer vectors for the host-side pieces that must match
the reference bit for bit: gen_synthetic traces, fit_quadratic, and
CPython's float sum().
"""

from __future__ import annotations

import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, str(Path(__file__).resolve().parent))

import pdsim  # noqa: E402
import pdsim.engine as engine_module  # noqa: E402
from scenarios import catalogue, catalogue_r2  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"

KIND = {"prefill_dispatch": 0, "decode_dispatch": 1, "flip": 2}
BRANCH = {
    name: i
    for i, name in enumerate(
        (
            "round-robin", "min-load", "alg1:t1", "alg1:t2", "alg1:flip", "alg1:fallback", "alg1:degenerate",
            "alg2:zero-transfer", "alg2:t1", "alg2:t2", "alg2:flip", "alg2:fallback", "alg2:forced-local",
        )
    )
}
TRIGGER = {name: i for i, name in enumerate(("alg1", "alg2", "monitor:tpot", "monitor:idle", "drained"))}
POOL = {"prefill": 0, "decode": 1, "p_to_d": 2, "d_to_p": 3}


def make(i, a, inp, out):
    return pdsim.TraceRequest(i, a, inp, out)


def encode_decisions(decisions, id_to_index):
    rows = []
    for d in decisions:
        if d["kind"] == "flip":
            code = TRIGGER[d["trigger"]] | (POOL[d["from"]] << 3) | (POOL[d["to"]] << 5)
            rows.append((d["time"], -1, d["instance"], 2, code))
        else:
            rows.append((d["time"], id_to_index[d["request_id"]], d["instance"], KIND[d["kind"]], BRANCH[d["branch"]]))
    arr = np.zeros(len(rows), dtype=[("time", "f8"), ("request", "i4"), ("instance", "i2"), ("kind", "u1"), ("code", "u1")])
    for k, r in enumerate(rows):
        arr[k] = r
    return arr


def run_one(sc):
    trace = sc["trace"]
    config = pdsim.config_from_values(sc["values"])
    scaled = pdsim.scale_trace(trace, sc["scale"]) if sc["scale"] != 1.0 else trace
    saved = engine_module.STALL_EVENT_LIMIT
    engine_module.STALL_EVENT_LIMIT = sc["stall_limit"]
    sim = engine_module._Simulation(scaled, config)
    t0 = time.perf_counter()
    try:
        result = sim.run()
        err = None
    except Exception as exc:  # noqa: BLE001
        result = None
        err = (type(exc).__name__, str(exc))
    finally:
        engine_module.STALL_EVENT_LIMIT = saved
    wall = time.perf_counter() - t0
    arrays = {
        "arrival": np.array([r.arrival for r in trace], dtype=np.float64),
        "input_len": np.array([r.input_len for r in trace], dtype=np.int32),
        "output_len": np.array([r.output_len for r in trace], dtype=np.int32),
        "ids": np.array([r.id for r in trace], dtype=np.int64),
        "predictor": np.array([sim.predictor.a2, sim.predictor.a1, sim.predictor.a0]),
        "max_tokens": np.array([sim.max_tokens], dtype=np.int64),
    }
    meta = dict(name=sc["name"], values=sc["values"], scale=sc["scale"], stall_limit=sc["stall_limit"],
                wall_s=wall, error=err, full=sc["full"])
    if result is not None:
        id_to_index = {r.id: i for i, r in enumerate(trace)}
        arrays["decisions"] = encode_decisions(result.decisions, id_to_index)
        recs = result.records
        arrays["first"] = np.array([r.token_times[0] for r in recs])
        arrays["last"] = np.array([r.token_times[-1] for r in recs])
        arrays["flags"] = np.array([r.ttft_ok | (r.tpot_ok << 1) | (r.slo_ok << 2) for r in recs], dtype=np.uint8)
        if not sc.get("compact"):
            arrays["ntok"] = np.array([len(r.token_times) for r in recs], dtype=np.int64)
            arrays["ttft"] = np.array([r.ttft for r in recs])
            arrays["tpot"] = np.array([r.tpot for r in recs])
        arrays["transitions"] = np.array([(i, POOL[a.value], POOL[b.value]) for i, a, b in result.transitions],
                                         dtype=np.int32).reshape(-1, 3)
        if sc["full"]:
            arrays["token_times"] = np.concatenate([np.array(r.token_times) for r in recs]) if recs else np.zeros(0)
            snaps = [(s.time, st.instance_id, POOL[st.pool.value], st.running_tokens, st.kv_used, st.queue_len,
                      st.pred_delay, math.nan if st.avg_interval is None else st.avg_interval,
                      st.prefill_count, st.decode_count)
                     for s in result.snapshots for st in s.per_instance]
            arrays["snapshots"] = np.array(snaps, dtype=[
                ("time", "f8"), ("instance", "i4"), ("pool", "i4"), ("running_tokens", "i4"), ("kv_used", "i4"),
                ("queue_len", "i4"), ("pred_delay", "f8"), ("avg_interval", "f8"), ("prefill_count", "i4"),
                ("decode_count", "i4")])
        if recs:
            s = pdsim.compute_metrics(recs, config.slo)
            meta["summary"] = s.to_dict()
        meta["n_events_hint"] = None
    return meta, arrays


def known_answers():
    kav = {}
    params = [
        dict(duration_s=50.0, base_rate=3.0, input_log_mean=math.log(300), input_log_sigma=0.5,
             output_log_mean=math.log(60), output_log_sigma=0.4, seed=11),
        dict(duration_s=30.0, base_rate=2.0, input_log_mean=math.log(1500), input_log_sigma=0.9,
             output_log_mean=math.log(40), output_log_sigma=0.8,
             bursts=(pdsim.BurstEpisode(5.0, 5.0, 5.0),), max_input=8000, max_output=1000, seed=101),
    ]
    traces = []
    for p in params:
        t = pdsim.gen_synthetic(pdsim.SyntheticParams(**p))
        traces.append(np.array([(r.arrival, r.input_len, r.output_len) for r in t]))
    b = pdsim.bundled_bursty_trace()
    r = pdsim.bundled_ramp_trace()
    fits = []
    for seed in range(4):
        for noise in (0.0, 0.02):
            for true in ((1e-7, 1e-4, 5e-3), (2e-8, 2e-5, 2e-3), (2e-7, 1e-4, 2e-3)):
                rng = np.random.default_rng(seed)
                grid = pdsim.default_profile_grid(16384, 16)
                f = pdsim.fit_quadratic(pdsim.profile_prefill(pdsim.PrefillCostParams(*true), grid, noise, rng))
                fits.append((seed, noise, *true, f.a2, f.a1, f.a0))
    rng = np.random.default_rng(99)
    sums = []
    vecs = []
    for k in range(200):
        n = int(rng.integers(1, 60))
        v = rng.standard_normal(n) * 10.0 ** rng.integers(-8, 9, size=n)
        if k % 5 == 0:
            v = np.abs(v)
        vecs.append(v)
        sums.append(sum(v.tolist()))
    lens = np.array([len(v) for v in vecs])
    return {
        "synthetic_0": traces[0],
        "synthetic_1": traces[1],
        "bursty": np.array([(x.arrival, x.input_len, x.output_len) for x in b]),
        "ramp": np.array([(x.arrival, x.input_len, x.output_len) for x in r]),
        "fits": np.array(fits),
        "pysum_values": np.concatenate(vecs),
        "pysum_lengths": lens,
        "pysum_results": np.array(sums),
        "max_tokens": np.array([
            pdsim.max_running_tokens(pdsim.DecodeCostParams(2e-5, 5e-3), 16000, 0.1),
            pdsim.max_running_tokens(pdsim.DecodeCostParams(1e-4, 4e-3), 3000, 0.1),
            pdsim.max_running_tokens(pdsim.DecodeCostParams(2e-5, 5e-3), 16000, 0.025),
        ]),
    }


def main():
    """GOLDEN_SET=r1 (default): the round-1 catalogue, rewriting index.json.
    GOLDEN_SET=r2[:c3,c4,c5,tie]: the BASELINE C3/C4/C5 scenarios and the
    burst-merge tie case (scenarios.catalogue_r2), merged into index.json by
    name; their fixtures are compact (no ttft/tpot/ntok arrays: those follow
    from first/last token times and output_len)."""
    OUT.mkdir(parents=True, exist_ok=True)
    include_slow = os.environ.get("GOLDEN_FAST") != "1"
    which = os.environ.get("GOLDEN_SET", "r1")
    index = []
    t_all = time.perf_counter()
    if which.startswith("r2"):
        parts = tuple(which.split(":", 1)[1].split(",")) if ":" in which else ("c3", "c4", "c5", "tie")
        scs = catalogue_r2(make, which=parts)
        for sc in scs:
            sc["compact"] = not sc["full"]
        old = json.loads((OUT / "index.json").read_text())
        names = {sc["name"] for sc in scs}
        index = [m for m in old["scenarios"] if m["name"] not in names]
    else:
        scs = catalogue(make, include_slow=include_slow)
    for sc in scs:
        meta, arrays = run_one(sc)
        fname = f"{sc['name']}.npz"
        np.savez_compressed(OUT / fname, **arrays)
        meta["file"] = fname
        index.append(meta)
        print(f"{sc['name']:28s} n={len(sc['trace']):5d} {meta['wall_s']:7.2f}s err={meta['error']}", flush=True)
    if not which.startswith("r2"):
        np.savez_compressed(OUT / "known_answers.npz", **known_answers())
    (OUT / "index.json").write_text(json.dumps(dict(
        generator="oracle/gen_golden.py",
        reference="/root/reference/pkg/src (pdsim)",
        python=sys.version.split()[0],
        numpy=np.__version__,
        scenarios=index,
    ), indent=1))
    print(f"total {time.perf_counter() - t_all:.1f}s")


if __name__ == "__main__":
    main()
