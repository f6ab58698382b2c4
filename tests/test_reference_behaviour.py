"""The reference's own behavioural contract (pkg/tests/test_engine.py and
test_acceptance.py), exercised through this package's
drop-in API on the CUDA evaluator: closed-form timelines, the FCFS
queueing recurrence, cadence of monitor ticks, determinism, token
conservation, strategy equivalences, the stall watchdog, and the
qualitative claims Arrow is built around."""

from __future__ import annotations

import dataclasses
import filecmp
import math

import numpy as np
import pytest

import paper_2505_11916_b200 as arrow
from paper_2505_11916_b200 import engine

pytestmark = pytest.mark.gpu

PREFILL = arrow.PrefillCostParams(2e-7, 1e-4, 2e-3)
DECODE = arrow.DecodeCostParams(1e-4, 4e-3)
TRANSFER = arrow.TransferParams(bandwidth=4e11, base_latency=1e-4, bytes_per_token=131072)


def cluster(n, *, strategy=arrow.Strategy.SLO_AWARE, split=(None, None), kv=16000, prefill=PREFILL, decode=DECODE,
            flips=True, seed=0):
    return arrow.RunConfig(
        instance_count=n,
        instance=arrow.InstanceConfig(kv, prefill, decode, TRANSFER),
        slo=arrow.SLOConfig(3.0, 0.1),
        scheduler=arrow.SchedulerConfig(strategy=strategy, enable_flips=flips),
        init_prefill=split[0],
        init_decode=split[1],
        seed=seed,
    )


SOLO = dict(split=(1, 0))


def synthetic(n=60, seed=11, rate=3.0, duration=20.0):
    p = arrow.SyntheticParams(duration, rate, math.log(300), 0.5, math.log(60), 0.4, seed=seed)
    return arrow.gen_synthetic(p)[:n]


def close(a, b, rel=1e-12):
    return abs(a - b) <= rel * max(abs(a), abs(b))


def test_one_request_on_one_instance():
    res = arrow.run([arrow.TraceRequest(0, 0.0, 300, 4)], cluster(1, **SOLO))
    t1 = arrow.predict_prefill_time(PREFILL, 300)
    d = arrow.decode_iter_time(DECODE, 1)
    rec = res.records[0]
    for got, exp in zip(rec.token_times, [t1, t1 + d, t1 + 2 * d, t1 + 3 * d]):
        assert close(got, exp)
    assert close(rec.tpot, d) and rec.slo_ok
    assert [x["branch"] for x in res.decisions] == ["alg1:t1", "alg2:forced-local"]
    assert res.transitions == []


def test_single_token_output_has_no_decode_phase():
    res = arrow.run([arrow.TraceRequest(0, 0.0, 200, 1)], cluster(1, **SOLO))
    assert len(res.records[0].token_times) == 1 and res.records[0].tpot == 0.0
    assert [x["kind"] for x in res.decisions] == ["prefill_dispatch"]


def test_long_prompt_is_chunked():
    res = arrow.run([arrow.TraceRequest(0, 0.0, 1300, 2)], cluster(1, **SOLO))
    t1 = sum(arrow.decode_iter_time(DECODE, c) for c in (512, 512, 276))
    assert close(res.records[0].ttft, t1)


def test_kv_transfer_shows_up_in_first_gap():
    res = arrow.run([arrow.TraceRequest(0, 0.0, 400, 3)],
                    cluster(2, strategy=arrow.Strategy.MINIMAL_LOAD, split=(1, 1)))
    t1 = arrow.predict_prefill_time(PREFILL, 400)
    d = arrow.decode_iter_time(DECODE, 1)
    mig = arrow.transfer_time(TRANSFER, 400)
    times = res.records[0].token_times
    assert close(times[1], t1 + mig + d) and close(times[2], t1 + mig + 2 * d)
    dec = [x for x in res.decisions if x["kind"] == "decode_dispatch"]
    assert len(dec) == 1 and dec[0]["instance"] == 1 and dec[0]["branch"] == "min-load"


def test_prefill_only_runs_follow_the_fcfs_recurrence():
    """Single-token outputs on one instance: a FCFS single server with
    quadratic service times (test_acceptance.py:78-111), 200 workloads."""
    rng = np.random.default_rng(7)
    base = arrow.default_run_config()
    cfg = dataclasses.replace(base, instance_count=1, init_prefill=1, init_decode=0,
                              instance=dataclasses.replace(base.instance, true_prefill=PREFILL))
    for _ in range(200):
        n = int(rng.integers(1, 51))
        arrivals = np.cumsum(rng.exponential(float(rng.uniform(0.001, 0.2)), size=n))
        lengths = rng.integers(1, 513, size=n)
        trace = [arrow.TraceRequest(i, float(a), int(L), 1) for i, (a, L) in enumerate(zip(arrivals, lengths))]
        res = arrow.run(trace, cfg)
        free = 0.0
        for req, rec in zip(trace, res.records):
            free = max(free, req.arrival) + arrow.predict_prefill_time(PREFILL, req.input_len)
            assert abs(rec.ttft - (free - req.arrival)) <= 1e-9


def test_monitor_ticks_every_period_until_done():
    cfg = cluster(1, **SOLO, prefill=arrow.PrefillCostParams(0.0, 0.01, 0.0), decode=arrow.DecodeCostParams(1e-9, 0.085))
    res = arrow.run([arrow.TraceRequest(0, 0.0, 100, 100)], cfg)
    assert [s.time for s in res.snapshots] == [float(t) for t in range(1, 11)]
    first = res.snapshots[0].per_instance[0]
    assert (first.running_tokens, first.decode_count, first.prefill_count) == (100, 1, 0)


def test_empty_trace():
    res = arrow.run([], cluster(2))
    assert res.records == [] and res.snapshots == [] and res.decisions == []


def test_deterministic_and_byte_identical_outputs(tmp_path):
    trace = arrow.bundled_bursty_trace()[:600]
    base = arrow.default_run_config()
    cfg = dataclasses.replace(base, instance=dataclasses.replace(
        base.instance, kv_capacity_tokens=3000, true_prefill=arrow.PrefillCostParams(2e-8, 2e-5, 2e-3)),
        init_prefill=4, init_decode=4)
    dirs = []
    for name in ("a", "b"):
        res = arrow.run(trace, cfg)
        arrow.write_outputs(res, cfg.slo, tmp_path / name)
        dirs.append(tmp_path / name)
    for f in ("requests.csv", "decisions.jsonl", "monitor.csv", "summary.json"):
        assert filecmp.cmp(dirs[0] / f, dirs[1] / f, shallow=False), f


def test_every_request_emits_output_len_tokens():
    trace = synthetic()
    res = arrow.run(trace, cluster(4, split=(2, 2)))
    assert len(res.records) == len(trace)
    for req, rec in zip(trace, res.records):
        assert len(rec.token_times) == req.output_len
        assert rec.token_times == sorted(rec.token_times) and rec.token_times[0] >= req.arrival


def test_slo_aware_without_flips_equals_minimal_load():
    trace = synthetic(n=120, duration=40.0)
    a = arrow.run(trace, cluster(4, split=(2, 2), flips=False))
    b = arrow.run(trace, cluster(4, strategy=arrow.Strategy.MINIMAL_LOAD, split=(2, 2)))
    pick = lambda r: [(d["kind"], d["request_id"], d["instance"]) for d in r.decisions if d["kind"] != "flip"]  # noqa: E731
    assert pick(a) == pick(b)
    assert [(r.ttft, r.tpot) for r in a.records] == [(r.ttft, r.tpot) for r in b.records]
    assert a.transitions == [] == b.transitions


def test_stall_watchdog(monkeypatch):
    monkeypatch.setattr(engine, "STALL_EVENT_LIMIT", 0)
    with pytest.raises(arrow.SimulationStallError, match="stalled"):
        arrow.run([arrow.TraceRequest(0, 0.0, 100, 4)], cluster(2))


def test_validation_errors():
    with pytest.raises(ValueError, match="sorted by arrival"):
        arrow.run([arrow.TraceRequest(0, 5.0, 10, 2), arrow.TraceRequest(1, 1.0, 10, 2)], cluster(2))
    with pytest.raises(ValueError, match="duplicate request id 7"):
        arrow.run([arrow.TraceRequest(7, 0.0, 10, 2), arrow.TraceRequest(7, 1.0, 10, 2)], cluster(2))
    with pytest.raises(ValueError, match="KV tokens"):
        arrow.run([arrow.TraceRequest(0, 0.0, 900, 200)], cluster(2, kv=1000))


def sweep_config(n, strategy):
    base = arrow.default_run_config()
    inst = dataclasses.replace(base.instance, kv_capacity_tokens=3000,
                               true_prefill=arrow.PrefillCostParams(2e-8, 2e-5, 2e-3))
    return dataclasses.replace(base, instance_count=n, instance=inst,
                               scheduler=arrow.SchedulerConfig(strategy=strategy), init_prefill=n // 2,
                               init_decode=n // 2)


def test_adaptive_sustains_higher_rate_than_static():
    """test_acceptance.py:308-332: max rate at 90 % attainment, adaptive >= 1.2x static."""
    trace = arrow.bundled_bursty_trace()
    grid = [6.0, 8.0, 9.0, 10.0, 11.0, 12.0]
    best = {}
    for s in (arrow.Strategy.SLO_AWARE, arrow.Strategy.MINIMAL_LOAD):
        best[s] = arrow.max_qualifying_rate(arrow.run_rate_sweep(trace, sweep_config(8, s), grid), 0.9)
    assert best[arrow.Strategy.MINIMAL_LOAD] is not None and best[arrow.Strategy.SLO_AWARE] is not None
    assert best[arrow.Strategy.SLO_AWARE] / best[arrow.Strategy.MINIMAL_LOAD] >= 1.2


def test_overload_resolves_toward_decode():
    reqs = [(0.1 * k, 200, 800) for k in range(80)] + [(5.0 + k / 30.0, 3000, 2) for k in range(90)]
    reqs.sort(key=lambda r: r[0])
    trace = [arrow.TraceRequest(i, a, il, ol) for i, (a, il, ol) in enumerate(reqs)]
    cfg = dataclasses.replace(arrow.default_run_config(), instance_count=4, init_prefill=2, init_decode=2)
    res = arrow.run(trace, cfg)
    flips = [d for d in res.decisions if d["kind"] == "flip"]
    assert any(f["to"] in ("p_to_d", "decode") for f in flips)
    assert not any(f["to"] in ("d_to_p", "prefill") for f in flips)


def test_prefill_load_peaks_before_decode_load():
    trace = arrow.scale_trace(arrow.bundled_ramp_trace(), 1.0 / 8.0)
    cfg = dataclasses.replace(arrow.default_run_config(), instance_count=8, init_prefill=4, init_decode=4,
                              scheduler=arrow.SchedulerConfig(strategy=arrow.Strategy.MINIMAL_LOAD))
    res = arrow.run(trace, cfg)
    pre = [(s.time, sum(x.prefill_count for x in s.per_instance if x.pool is arrow.PoolKind.PREFILL))
           for s in res.snapshots]
    dec = [(s.time, sum(x.decode_count for x in s.per_instance if x.pool is arrow.PoolKind.DECODE))
           for s in res.snapshots]
    tp, pp = max(pre, key=lambda x: x[1])
    td, pd = max(dec, key=lambda x: x[1])
    assert pp >= 3 and pd >= 50 and tp < td


def test_attainment_grows_with_cluster_size():
    trace = arrow.bundled_bursty_trace()
    att = [arrow.run_rate_sweep(trace, sweep_config(n, arrow.Strategy.SLO_AWARE), [6.0])[0][1].attainment
           for n in (2, 4, 8)]
    assert att[0] <= att[1] <= att[2]


def test_sweep_equals_individual_runs():
    """One batched launch over a rate grid == per-rate drop-in runs + host
    compute_metrics (report.py:77-91 semantics), bit for bit."""
    trace = arrow.bundled_bursty_trace()[:800]
    cfg = sweep_config(8, arrow.Strategy.SLO_AWARE)
    rates = [4.0, 7.0, 10.0]
    swept = arrow.run_rate_sweep(trace, cfg, rates)
    base = arrow.native_rate(trace)
    for rate, summary in swept:
        res = arrow.run(arrow.scale_trace(trace, base / rate), cfg)
        assert summary == arrow.compute_metrics(res.records, cfg.slo)
