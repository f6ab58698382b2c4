"""CUDA evaluator parity (needs a B200): every golden scenario of the real
reference, bit for bit, and seeded random sweeps against the CPU oracle."""

from __future__ import annotations

import numpy as np
import pytest

import harness as H
from paper_2505_11916_b200 import _abi
from paper_2505_11916_b200._buffers import OutputSpec
from paper_2505_11916_b200._compile import Scenario, compile_batch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def evaluator():
    from paper_2505_11916_b200._backend import CudaEvaluator

    return CudaEvaluator()


def _runnable():
    out = []
    for meta in H.golden_index():
        if meta["error"] and meta["error"][0] == "ValueError":
            continue
        out.append((meta, H.golden_arrays(meta)))
    return out


def test_golden_scenarios_bit_exact(evaluator):
    """All reference-generated scenarios, batched by watchdog limit."""
    items = _runnable()
    by_limit: dict[int, list] = {}
    for m, a in items:
        by_limit.setdefault(m["stall_limit"], []).append((m, a))
    checked = 0
    for group in by_limit.values():
        cb = H.compile_golden(group)
        hb = evaluator.execute(cb, H.spec_for(group))
        for s, (m, a) in enumerate(group):
            H.check_vs_golden(m, a, hb, s)
            checked += 1
    assert checked == len(items)


def _random_scenarios(seed: int, count: int):
    import sys

    sys.path.insert(0, str(H.ROOT / "oracle"))
    import scenarios as S
    from paper_2505_11916_b200.config import config_from_values
    from paper_2505_11916_b200.core import TraceRequest

    rng = np.random.default_rng(seed)
    traces = [S.bursty(TraceRequest)[:600], S.small_trace(TraceRequest, n=200, duration=80.0), S.ramp(TraceRequest)]
    out = []
    for k in range(count):
        tr = traces[k % len(traces)]
        N = int(rng.integers(2, 17))
        strat = ["slo-aware", "slo-aware", "minimal-load", "round-robin"][int(rng.integers(0, 4))]
        n_p = int(rng.integers(1, N))
        v = S.cfg(
            instances=N, init_prefill=n_p, init_decode=N - n_p, strategy=strat,
            enable_flips=bool(rng.integers(0, 4) > 0),
            kv_capacity_tokens=int(rng.choice([5000, 8000, 16000])),
            chunk_budget=int(rng.choice([256, 512])),
            theta_d=float(rng.choice([0.25, 0.5, 1.0])), theta_busy=float(rng.choice([0.5, 0.75, 1.0])),
            tpot_breach_duration_s=float(rng.choice([1.0, 2.0, 4.0])),
            a2=2e-8, a1=2e-5, a0=2e-3,
        )
        rate = float(rng.uniform(0.5, 3.0)) * N
        out.append(Scenario(tr, config_from_values(v), S.rate_scale(tr, rate), k))
    return out


@pytest.mark.parametrize("seed", [1, 2])
def test_random_sweep_matches_oracle(evaluator, seed):
    scs = _random_scenarios(seed, 96)
    cb = compile_batch(scs, 20000)
    spec = OutputSpec(requests=True)
    got = evaluator.execute(cb, spec)
    exp = H.run_oracle(cb, spec, threads=0)
    for s in range(cb.n):
        g, e = got.summaries[s], exp.summaries[s]
        assert int(g["status"]) == int(e["status"]), (s, g["status"], e["status"])
        for f in ("n_completed", "n_ok", "n_flips", "n_events", "n_iterations", "n_decisions", "n_ticks",
                  "decision_hash"):
            assert int(g[f]) == int(e[f]), (s, f, g[f], e[f])
        for f in ("stall_time", "attainment", "p90_ttft", "p90_tpot", "mean_ttft", "mean_tpot", "goodput", "span"):
            H.assert_same_f64([g[f]], [e[f]], f"scenario {s} {f}")
    H.assert_same_f64(got.req_first, exp.req_first, "first")
    for s in range(cb.n):
        if int(exp.summaries[s]["status"]) == _abi.OK:   # stalled runs raise; partial records unobserved
            sl = got.req_slice(s)
            H.assert_same_f64(got.req_last[sl], exp.req_last[sl], f"scenario {s} last")
    np.testing.assert_array_equal(got.req_prefill, exp.req_prefill)
    np.testing.assert_array_equal(got.req_decode, exp.req_decode)
    assert (got.summaries["status"] == _abi.OK).sum() > 0


def test_large_clusters_two_instances_per_lane(evaluator):
    """N > 32 puts two instances on each lane (register slots 0 and 1):
    C4-style clusters of 33-64 instances against the CPU oracle."""
    import sys

    sys.path.insert(0, str(H.ROOT / "oracle"))
    import scenarios as S
    from paper_2505_11916_b200.config import config_from_values
    from paper_2505_11916_b200.core import TraceRequest

    trace = S.synthetic(TraceRequest, 600.0, 4.0, np.log(420.0), 0.55, np.log(130.0), 0.5,
                        ((100.0, 60.0, 5.0), (300.0, 90.0, 4.0)), 3500, 900, 3)[:2000]
    scs = []
    for k, (N, strat, td, rate_per) in enumerate([(33, "slo-aware", 0.5, 1.25), (48, "slo-aware", 0.25, 2.5),
                                                   (64, "slo-aware", 1.0, 2.5), (40, "minimal-load", 0.5, 2.0),
                                                   (64, "round-robin", 0.5, 1.0), (64, "slo-aware", 0.75, 4.0)]):
        v = S.cfg(instances=N, init_prefill=N // 2, init_decode=N - N // 2, strategy=strat, theta_d=td,
                  kv_capacity_tokens=6000)
        scs.append(Scenario(trace, config_from_values(v), S.rate_scale(trace, rate_per * N), k))
    cb = compile_batch(scs, 500_000)
    assert cb.sizes["max_instances"] == 64
    spec = OutputSpec(requests=True, decisions=True)
    got = evaluator.execute(cb, spec)
    exp = H.run_oracle(cb, spec, threads=0)
    for s in range(cb.n):
        g, e = got.summaries[s], exp.summaries[s]
        for f in ("status", "n_completed", "n_ok", "n_flips", "n_events", "n_iterations", "n_decisions",
                  "decision_hash"):
            assert int(g[f]) == int(e[f]), (s, f, g[f], e[f])
        if int(e["status"]) == _abi.OK:
            H.assert_same_decisions(got.decisions_of(s), exp.decisions_of(s))
            sl = got.req_slice(s)
            H.assert_same_f64(got.req_last[sl], exp.req_last[sl], f"scenario {s} last")


@pytest.mark.parametrize("build", ["latency", "throughput"])
def test_both_kernel_builds_bit_exact(build):
    """The latency build (unbounded registers) and the occupancy build
    (3 blocks/SM) are the same source under different launch bounds; both,
    forced regardless of batch size, reproduce the golden scenarios and the
    oracle's random sweep (IPL 1 and 2)."""
    from paper_2505_11916_b200._backend import CudaEvaluator

    ev = CudaEvaluator(build=build)
    items = _runnable()
    by_limit: dict[int, list] = {}
    for m, a in items:
        by_limit.setdefault(m["stall_limit"], []).append((m, a))
    for group in by_limit.values():
        cb = H.compile_golden(group)
        hb = ev.execute(cb, H.spec_for(group))
        for s, (m, a) in enumerate(group):
            H.check_vs_golden(m, a, hb, s)
    scs = _random_scenarios(7, 48)
    cb = compile_batch(scs, 20000)
    got = ev.execute(cb, OutputSpec(requests=True))
    exp = H.run_oracle(cb, OutputSpec(requests=True), threads=0)
    for s in range(cb.n):
        for f in ("status", "n_completed", "n_ok", "n_flips", "n_events", "n_decisions", "decision_hash"):
            assert int(got.summaries[s][f]) == int(exp.summaries[s][f]), (build, s, f)
    np.testing.assert_array_equal(got.req_prefill, exp.req_prefill)


def test_lockstep_instances_match_oracle(evaluator):
    """Simultaneous identical requests on identical instances (exact event
    time ties), both kernel builds, against the CPU oracle."""
    from paper_2505_11916_b200._backend import CudaEvaluator

    cb = compile_batch(H.lockstep_scenarios(), 500_000)
    spec = OutputSpec(requests=True)
    exp = H.run_oracle(cb, spec)
    for ev in (evaluator, CudaEvaluator(build="throughput")):
        H.assert_same_run(ev.execute(cb, spec), exp, cb.n)
