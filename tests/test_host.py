"""Host-side logic of the drop-in layer (no GPU): configuration, validation
and error behaviour mirroring the reference, and assembly of the
reference's Python objects (records with full token_times, decision dicts,
snapshots, stall messages) from raw evaluator outputs — fed here by the CPU
oracle, which writes the same output buffers as the CUDA kernel."""

from __future__ import annotations

import math

import numpy as np
import pytest

import harness as H
import paper_2505_11916_b200 as arrow
from paper_2505_11916_b200 import _results
from paper_2505_11916_b200._compile import emission_capacity

INDEX = {m["name"]: m for m in H.golden_index()}


def _oracle(name, tokens=False):
    meta = INDEX[name]
    arrays = H.golden_arrays(meta)
    cb = H.compile_golden([(meta, arrays)])
    return meta, arrays, cb, H.run_oracle(cb, tokens=tokens)


@pytest.mark.parametrize("name", ["single_request", "chunked_prefill", "migration_gap", "small_arrow_2_2",
                                  "overload_flips", "c1_rate4", "determinism_600"])
def test_token_times_rebuilt_from_iteration_log(name):
    """Full token_times from first-token time + the decode instance's
    iteration log equal the reference's recorded token lists."""
    meta, arrays, cb, hb = _oracle(name)
    entry = cb.table.entries[0]
    recs = _results.records(hb, 0, entry.arrival * cb.scenarios["arrival_scale"][0], entry.ids,
                            arrow.config_from_values(meta["values"]).slo)
    got = np.concatenate([np.array(r.token_times) for r in recs])
    H.assert_same_f64(got, arrays["token_times"], "token times")
    summary = arrow.compute_metrics(recs, arrow.config_from_values(meta["values"]).slo)
    for k in H.SUMMARY_KEYS:
        assert H.bits(getattr(summary, k)) == H.bits(meta["summary"][k]), k


def test_decision_dicts_and_transitions():
    meta, arrays, cb, hb = _oracle("overload_flips")
    dec = _results.decision_dicts(hb, 0, cb.table.entries[0].ids)
    kinds = {d["kind"] for d in dec}
    assert kinds == {"prefill_dispatch", "decode_dispatch", "flip"}
    flips = [d for d in dec if d["kind"] == "flip"]
    assert list(flips[0]) == ["time", "kind", "instance", "from", "to", "trigger"]
    disp = next(d for d in dec if d["kind"] != "flip")
    assert list(disp) == ["time", "kind", "request_id", "instance", "branch"]
    tr = _results.transitions(dec)
    assert [(i, a.value, b.value) for i, a, b in tr] == [
        (int(i), arrow.core.POOL_BY_CODE[a].value, arrow.core.POOL_BY_CODE[b].value) for i, a, b in arrays["transitions"]
    ]
    # overload resolution favours decode (test_acceptance.py:352-380)
    assert all(f["to"] in ("p_to_d", "decode") for f in flips) and flips


def test_snapshot_assembly():
    meta, arrays, cb, hb = _oracle("monitor_cadence")
    snaps = _results.snapshots(hb, 0)
    assert [s.time for s in snaps] == [float(t) for t in range(1, 11)]
    first = snaps[0].per_instance[0]
    assert first.running_tokens == 100 and first.decode_count == 1 and first.prefill_count == 0
    assert snaps[0].pool_counts()[arrow.PoolKind.PREFILL] == 1


def test_stall_message_matches_reference():
    for name in ("stall_limit_zero", "c2_coloc_r20_stall"):
        meta, arrays, cb, hb = _oracle(name)
        with pytest.raises(arrow.SimulationStallError) as exc:
            _results.raise_for_status(hb, 0)
        assert str(exc.value) == meta["error"][1]


def test_config_validation_mirrors_reference():
    mk = lambda **kw: arrow.config_from_values({**arrow.config.DEFAULTS, **kw})  # noqa: E731
    with pytest.raises(ValueError, match="instance_count"):
        mk(instances=0)
    with pytest.raises(ValueError, match="does not partition"):
        mk(instances=4, init_prefill=5, init_decode=-1)
    with pytest.raises(ValueError, match="static strategies"):
        mk(instances=4, strategy="minimal-load", init_prefill=4, init_decode=0)
    with pytest.raises(ValueError, match="theta_d"):
        mk(theta_d=0.0)
    assert mk(instances=5).initial_split() == (3, 2)
    assert mk(instances=4, init_prefill=1).initial_split() == (1, 3)
    assert mk(instances=4, init_decode=1).initial_split() == (3, 1)


def test_config_text_parsing():
    values = arrow.parse_config_text("# c\ninstances = 4\ninit_prefill = 3  # x\nstrategy = minimal-load\n"
                                     "enable_flips = false\ntpot_slo = 0.25\n")
    cfg = arrow.config_from_values(values)
    assert cfg.instance_count == 4 and cfg.initial_split() == (3, 1)
    assert cfg.scheduler.strategy is arrow.Strategy.MINIMAL_LOAD and cfg.scheduler.enable_flips is False
    with pytest.raises(ValueError, match=r"cfg:2: unknown config key 'instnaces'"):
        arrow.parse_config_text("seed = 1\ninstnaces = 4\n", source="cfg")
    with pytest.raises(ValueError, match=r"cfg:1: bad value for 'seed'"):
        arrow.parse_config_text("seed = lots\n", source="cfg")
    with pytest.raises(ValueError, match=r"cfg:1: expected `key = value`"):
        arrow.parse_config_text("just some words\n", source="cfg")


def test_trace_validation_errors():
    from paper_2505_11916_b200._compile import Scenario, compile_batch

    cfg = arrow.default_run_config()
    bad = [
        ([arrow.TraceRequest(0, 5.0, 10, 2), arrow.TraceRequest(1, 1.0, 10, 2)], "sorted by arrival"),
        ([arrow.TraceRequest(7, 0.0, 10, 2), arrow.TraceRequest(7, 1.0, 10, 2)], "duplicate request id 7"),
        ([arrow.TraceRequest(0, 0.0, 16000, 200)], "needs 16200 KV tokens"),
    ]
    for trace, msg in bad:
        with pytest.raises(ValueError, match=msg):
            compile_batch([Scenario(trace, cfg)], 500_000)


def test_scale_trace_and_rates():
    trace = [arrow.TraceRequest(0, 2.0, 10, 2), arrow.TraceRequest(1, 4.0, 20, 3)]
    assert [r.arrival for r in arrow.scale_trace(trace, 0.5)] == [1.0, 2.0]
    assert trace[0].arrival == 2.0
    with pytest.raises(ValueError, match="scale factor"):
        arrow.scale_trace(trace, 0.0)
    assert arrow.native_rate(trace) == 0.5
    with pytest.raises(ValueError, match="empty rate grid"):
        arrow.run_rate_sweep(trace, arrow.default_run_config(), [])
    with pytest.raises(ValueError, match="rates must be positive"):
        arrow.run_rate_sweep(trace, arrow.default_run_config(), [1.0, -2.0])


def test_percentile_and_max_rate():
    vals = [float(i) for i in range(1, 11)]
    assert arrow.percentile_nearest_rank(vals, 0.9) == 9.0
    assert arrow.percentile_nearest_rank([42.0], 0.9) == 42.0
    S = arrow.RunSummary
    res = [(r, S(a, 0, 0, 0, 0, 0, 1, 1.0)) for r, a in ((1.0, 0.95), (2.0, 0.91), (3.0, 0.5))]
    assert arrow.max_qualifying_rate(res, 0.9) == 2.0
    assert arrow.max_qualifying_rate(res, 0.99) is None


def test_emission_ring_bound_covers_window():
    cfg = arrow.default_run_config()
    cap = emission_capacity(cfg)
    # four windows of 5 s / shortest iteration (b1 + b0 = 5.02 ms): 4 x ~1000 emissions
    assert 3960 < cap < 4400
    assert emission_capacity(arrow.config_from_values({**arrow.config.DEFAULTS, "a0": 0.0, "a1": 0.0, "a2": 0.0})) \
        == 1 << 16


def test_output_writers_round_trip(tmp_path):
    meta, arrays, cb, hb = _oracle("small_arrow_2_2")
    entry = cb.table.entries[0]
    cfg = arrow.config_from_values(meta["values"])
    recs = _results.records(hb, 0, entry.arrival, entry.ids, cfg.slo)
    dec = _results.decision_dicts(hb, 0, entry.ids)
    result = arrow.RunResult(recs, _results.snapshots(hb, 0), dec, _results.transitions(dec))
    paths = arrow.write_outputs(result, cfg.slo, tmp_path)
    rows = arrow.report.read_request_csv(paths["requests"])
    assert [r["ttft_s"] for r in rows] == [r.ttft for r in recs]
    assert paths["decisions"].read_text().count("\n") == len(dec)
    assert math.isfinite(float(paths["summary"].read_text().split('"attainment": ')[1].split(",")[0]))


def test_unbounded_max_batch_and_transfer_product_limits():
    """max_batch_requests above int32 (the reference accepts e.g. 10**10 as
    unbounded) compiles to min(max_batch, chunk_budget), the only value the
    batch former uses (instance.py:183); a prompt * bytes_per_token product
    that could overflow int64 on the device is rejected up front."""
    import dataclasses

    from paper_2505_11916_b200._compile import Scenario, compile_batch
    from paper_2505_11916_b200.config import default_run_config
    from paper_2505_11916_b200.core import TraceRequest

    base = default_run_config()
    trace = [TraceRequest(0, 0.0, 100, 5), TraceRequest(1, 1.0, 100, 5)]
    cfg = dataclasses.replace(base, instance=dataclasses.replace(base.instance, max_batch_requests=10**10))
    cb = compile_batch([Scenario(trace, cfg, 1.0)], 500_000)
    assert int(cb.scenarios["max_batch"][0]) == base.instance.chunk_budget
    big = dataclasses.replace(base.instance.transfer, bytes_per_token=1 << 50)
    cfg = dataclasses.replace(base, instance=dataclasses.replace(base.instance, transfer=big))
    with pytest.raises(ValueError, match="bytes_per_token"):
        compile_batch([Scenario(trace, cfg, 1.0)], 500_000)
