"""Device workload generator on the B200.

Bit-exact against the real reference's gen_synthetic (golden catalogue),
against the numpy host generator on seeded random parameter sets and on a
multi-seed batch, and end to end: a sweep over device-resident traces gives
the same per-scenario summaries (including the decision-stream digest) as
the same traces shipped from the host.
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np
import pytest

import harness as H
import synth_harness as SH
from paper_2505_11916_b200 import _abi

pytestmark = pytest.mark.gpu


def _arrays(dt):
    a, i, o = dt.arrays()
    return a, i.astype(np.int64), o.astype(np.int64)


def test_golden_catalogue_bit_exact():
    import paper_2505_11916_b200 as arrow

    entries = SH.golden_entries()
    ts = arrow.gen_synthetic_batch([p for _, p, _ in entries])
    for (name, _p, exp), dt in zip(entries, ts):
        SH.assert_trace_equal(name, _arrays(dt), exp)
        assert dt.n == len(exp[0])
        if dt.n:
            assert SH.isclose_bits(dt.first_arrival, float(exp[0][0]))
            assert SH.isclose_bits(dt.last_arrival, float(exp[0][-1]))
            assert dt.max_kv == int((exp[1] + exp[2]).max())
    # to_host() is the reference's list[TraceRequest]
    trace = ts[0].to_host()
    assert trace[5].id == 5 and trace[5].arrival == float(entries[0][2][0][5])


def test_random_params_bit_exact():
    import paper_2505_11916_b200 as arrow

    rng = np.random.default_rng(11916)
    params = [SH.random_params(rng) for _ in range(160)]
    ts = arrow.gen_synthetic_batch(params)
    for k, (p, dt) in enumerate(zip(params, ts)):
        SH.assert_trace_equal(f"random[{k}]", _arrays(dt), SH.host_trace_arrays(p))


def test_multi_seed_batch():
    """4096 seeds of the bursty workload: a sample is compared with numpy,
    every trace is checked for the generator's invariants."""
    import paper_2505_11916_b200 as arrow

    base = SH.params_of(dict(SH.catalogue())["bursty"])
    params = [replace(base, duration_s=60.0, seed=s) for s in range(4096)]
    ts = arrow.gen_synthetic_batch(params)
    for k in range(0, 4096, 257):
        SH.assert_trace_equal(f"seed {k}", _arrays(ts[k]), SH.host_trace_arrays(params[k]))
    arr = ts.arrival.cpu().numpy()
    inp = ts.input_len.cpu().numpy()
    out = ts.output_len.cpu().numpy()
    for k in range(4096):
        o, n = int(ts.offsets[k]), int(ts.counts[k])
        a = arr[o : o + n]
        assert n > 0 and (np.diff(a) >= 0).all() and a[0] >= 0 and a[-1] < 60.0
        assert inp[o : o + n].min() >= 1 and inp[o : o + n].max() <= base.max_input
        assert out[o : o + n].min() >= 1 and out[o : o + n].max() <= base.max_output
        assert int(inp[o : o + n].sum()) == int(ts.results["sum_input"][k])


def test_capacity_retry(monkeypatch):
    import paper_2505_11916_b200 as arrow
    from paper_2505_11916_b200 import device_traces

    monkeypatch.setattr(device_traces, "_capacity", lambda p: 7)
    entries = SH.golden_entries()[:6]
    ts = arrow.gen_synthetic_batch([p for _, p, _ in entries])
    assert (ts.results["status"] == _abi.SYNTH_OK).all()
    for (name, _p, exp), dt in zip(entries, ts):
        SH.assert_trace_equal(name, _arrays(dt), exp)


def test_reference_errors():
    import paper_2505_11916_b200 as arrow

    p = SH.params_of(dict(SH.catalogue())["small"])
    for bad, field in ((replace(p, max_input=0), "input_len"), (replace(p, max_output=-3), "output_len")):
        with pytest.raises(ValueError) as host:
            arrow.gen_synthetic(bad)
        with pytest.raises(ValueError) as dev:
            arrow.gen_synthetic_batch([bad])
        assert str(host.value) == str(dev.value) and field in str(dev.value)
    huge = replace(p, input_log_mean=800.0)
    with pytest.raises(OverflowError) as host:
        arrow.gen_synthetic(huge)
    with pytest.raises(OverflowError) as dev:
        arrow.gen_synthetic_batch([huge])
    assert str(host.value) == str(dev.value)
    assert len(arrow.gen_synthetic_batch([replace(p, duration_s=0.0)])[0]) == 0


def test_sweep_on_device_traces_matches_host_traces():
    """Scenarios over generated traces read in place == the same traces
    uploaded from the host (all summary fields, bitwise)."""
    import paper_2505_11916_b200 as arrow
    from paper_2505_11916_b200._compile import Scenario

    base = SH.params_of(dict(SH.catalogue())["bursty"])
    params = [replace(base, duration_s=90.0, seed=s) for s in (1, 2, 3, 4)]
    ts = arrow.gen_synthetic_batch(params)
    hosts = [dt.to_host() for dt in ts]
    import scenarios as S

    cfg = arrow.config_from_values(S.cfg(instances=8, kv_capacity_tokens=3000, a2=2e-8, a1=2e-5, a0=2e-3))
    coloc = replace(cfg, scheduler=replace(cfg.scheduler, enable_flips=False))
    dev_sc, host_sc = [], []
    for k, dt in enumerate(ts):
        for rate in (6.0, 12.0, 20.0):
            for c in (cfg, coloc):
                s = arrow.native_rate(dt) / rate
                assert s == arrow.native_rate(hosts[k]) / rate
                dev_sc.append(Scenario(dt, c, s))
                host_sc.append(Scenario(hosts[k], c, s))
    hd = arrow.evaluate_scenarios(dev_sc)
    hh = arrow.evaluate_scenarios(host_sc)
    fields = [f for f in _abi.SUMMARY_DTYPE.names if f not in ("cycles", "reserved")]  # SM clock profile
    for f in fields:
        assert hd.summaries[f].tobytes() == hh.summaries[f].tobytes(), f
    # full per-request outputs through run() on a device trace
    small = arrow.gen_synthetic_batch([replace(base, duration_s=40.0, seed=77)])[0]
    r_dev = arrow.run(small, cfg)
    r_host = arrow.run(small.to_host(), cfg)
    assert r_dev.decisions == r_host.decisions
    assert [r.token_times for r in r_dev.records] == [r.token_times for r in r_host.records]
    # rate sweep through the drop-in report API
    assert arrow.run_rate_sweep(ts[0], cfg, [5.0, 10.0]) == arrow.run_rate_sweep(hosts[0], cfg, [5.0, 10.0])


def test_multi_seed_sweep_vs_oracle(monkeypatch):
    """A multi-seed sweep the way the device generator is meant to be used:
    24 seeds generated on the GPU, each evaluated in place under Arrow /
    static PD / colocated at two rates; every summary field and the
    decision-stream digest equal the CPU oracle run on the same traces."""
    import paper_2505_11916_b200 as arrow
    import scenarios as S
    from paper_2505_11916_b200._buffers import OutputSpec
    from paper_2505_11916_b200._compile import Scenario, compile_batch

    monkeypatch.setattr(arrow.engine, "STALL_EVENT_LIMIT", 20000)  # read per call, like engine.py:283
    base = SH.params_of(dict(SH.catalogue())["bursty"])
    ts = arrow.gen_synthetic_batch([replace(base, duration_s=120.0, seed=9000 + s) for s in range(24)])
    arrow_cfg = arrow.config_from_values(S.cfg(instances=8, kv_capacity_tokens=4400, a2=2e-8, a1=2e-5, a0=2e-3))
    static_cfg = replace(arrow_cfg, scheduler=replace(arrow_cfg.scheduler, strategy=arrow.Strategy.MINIMAL_LOAD))
    coloc = arrow.config_from_values(S.cfg(instances=8, init_prefill=8, init_decode=0, enable_flips=False,
                                           kv_capacity_tokens=4400, a2=2e-8, a1=2e-5, a0=2e-3))
    dev, host = [], []
    hosts = [dt.to_host() for dt in ts]
    for k, dt in enumerate(ts):
        for cfg in (arrow_cfg, static_cfg, coloc):
            for rate in (8.0, 20.0):
                scale = arrow.native_rate(dt) / rate
                dev.append(Scenario(dt, cfg, scale))
                host.append(Scenario(hosts[k], cfg, scale))
    got = arrow.evaluate_scenarios(dev)
    exp = H.run_oracle(compile_batch(host, 20000), OutputSpec(), threads=0)
    for s in range(len(dev)):
        g, e = got.summaries[s], exp.summaries[s]
        for f in ("status", "n_completed", "n_ok", "n_flips", "n_events", "n_iterations", "n_decisions", "n_ticks",
                  "decision_hash"):
            assert int(g[f]) == int(e[f]), (s, f, g[f], e[f])
        for f in ("stall_time", "attainment", "p90_ttft", "p90_tpot", "mean_ttft", "mean_tpot", "goodput", "span"):
            H.assert_same_f64([g[f]], [e[f]], f"scenario {s} {f}")
    assert (got.summaries["status"] == _abi.OK).sum() > len(dev) // 2
