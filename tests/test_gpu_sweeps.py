"""BASELINE sweeps on the B200 against the CPU oracle (needs a GPU).

The oracle is pinned to the real reference on the C3/C4/C5 golden fixtures
(test_oracle_golden.py); here the CUDA evaluator runs seeded samples of the
full C3, C4 and C5 sweeps (workloads.py, the exact scenarios bench.py
times) and every per-scenario summary field, the decision-stream digest and
every request's first/last token time and dispatch targets must equal the
oracle's bit for bit, stalled scenarios included."""

from __future__ import annotations

import numpy as np
import pytest

import harness as H
from paper_2505_11916_b200 import _abi, engine
from paper_2505_11916_b200 import workloads as W
from paper_2505_11916_b200._buffers import OutputSpec
from paper_2505_11916_b200._compile import compile_batch, dispatch_order

pytestmark = pytest.mark.gpu

SUMMARY_INT = ("status", "n_completed", "n_ok", "n_flips", "n_events", "n_iterations", "n_decisions", "n_ticks",
               "decision_hash")
SUMMARY_F64 = ("stall_time", "attainment", "p90_ttft", "p90_tpot", "mean_ttft", "mean_tpot", "goodput", "span")


@pytest.fixture(scope="module")
def evaluator():
    from paper_2505_11916_b200._backend import CudaEvaluator

    return CudaEvaluator()


def _compare(got, exp, n):
    for f in SUMMARY_INT:
        g, e = got.summaries[f], exp.summaries[f]
        bad = np.nonzero(g != e)[0]
        assert bad.size == 0, f"{f}: {bad.size} scenarios differ, first {bad[0]}: {g[bad[0]]} vs {e[bad[0]]}"
    for f in SUMMARY_F64:
        H.assert_same_f64(got.summaries[f], exp.summaries[f], f)
    H.assert_same_f64(got.req_first, exp.req_first, "first")
    np.testing.assert_array_equal(got.req_prefill, exp.req_prefill)
    np.testing.assert_array_equal(got.req_decode, exp.req_decode)
    for s in range(n):
        if int(exp.summaries[s]["status"]) == _abi.OK:   # stalled runs raise; partial records unobserved
            sl = got.req_slice(s)
            H.assert_same_f64(got.req_last[sl], exp.req_last[sl], f"scenario {s} last")


def _run(evaluator, scenarios):
    cb = compile_batch(scenarios, engine.STALL_EVENT_LIMIT)
    spec = OutputSpec(requests=True)
    got = evaluator.execute(cb, spec, dispatch_order(cb))
    exp = H.run_oracle(cb, spec, threads=0)
    _compare(got, exp, cb.n)
    return got


def test_c5_sample_of_2048_matches_oracle(evaluator):
    """2 048 seeded C5 scenario ids (all traces, rates, policies, N up to 32,
    threshold axes), occupancy build (multi-wave), 500 000-event watchdog."""
    ids = np.sort(np.random.default_rng(2048).choice(98304, size=2048, replace=False))
    got = _run(evaluator, W.c5(ids))
    assert (got.summaries["status"] == _abi.OK).sum() > 2000


def test_c4_sample_matches_oracle(evaluator):
    """C4: 10 000-request Arrow runs on 16-64 instances (two instances per lane
    above 32), threshold ablation axes."""
    ids = np.sort(np.random.default_rng(4).choice(1080, size=96, replace=False))
    scs = W.c4(ids)
    assert max(s.config.instance_count for s in scs) == 64
    _run(evaluator, scs)


def test_c3_sample_matches_oracle(evaluator):
    """C3: code- and conversation-like traces over the TTFT x TPOT SLO grid
    (Arrow re-simulated per SLO point: thresholds and token cap follow)."""
    ids = np.sort(np.random.default_rng(3).choice(1920, size=192, replace=False))
    _run(evaluator, W.c3(ids))


def _adversarial_predictor_scenarios(seed: int, count: int):
    """Heavy profiling noise (profile_noise 1-10) fits predictors with
    negative a2 / a1 / a0: predicted prefill terms of mixed sign that cancel
    in the delay fold, the case the delay-interval bound must survive."""
    import sys

    sys.path.insert(0, str(H.ROOT / "oracle"))
    import scenarios as S
    from paper_2505_11916_b200._compile import Scenario
    from paper_2505_11916_b200.config import config_from_values
    from paper_2505_11916_b200.core import TraceRequest

    rng = np.random.default_rng(seed)
    tr = S.bursty(TraceRequest)[:400]
    out = []
    for k in range(count):
        N = int(rng.integers(2, 13))
        n_p = int(rng.integers(1, N))
        v = S.cfg(instances=N, init_prefill=n_p, init_decode=N - n_p,
                  strategy=["slo-aware", "slo-aware", "minimal-load"][k % 3],
                  profile_noise=float(rng.choice([1.0, 3.0, 10.0])), seed=int(rng.integers(0, 50)),
                  kv_capacity_tokens=int(rng.choice([3000, 8000])), a2=2e-8, a1=2e-5, a0=2e-3,
                  ttft_slo=float(rng.choice([0.5, 3.0])))
        out.append(Scenario(tr, config_from_values(v), S.rate_scale(tr, float(rng.uniform(0.5, 3.0)) * N), k))
    return out


def test_adversarial_predictor_sweep_matches_oracle(evaluator):
    cb = compile_batch(_adversarial_predictor_scenarios(11, 256), 20000)
    spec = OutputSpec(requests=True)
    _compare(evaluator.execute(cb, spec), H.run_oracle(cb, spec, threads=0), cb.n)


# Whole sweeps against the REAL reference: tests/golden/digest_<set>.npz
# (oracle/gen_golden_digest.py) holds, for every scenario of C3 (1 920) and
# C4 (1 080) and 512 seeded C5 ids, the reference's status / stall time,
# every RunSummary field and the FNV-1a digest of its decision stream.
DIGEST_FIELDS = (("attainment", "attainment"), ("p90_ttft", "p90_ttft"), ("p90_tpot", "p90_tpot"),
                 ("mean_ttft", "mean_ttft"), ("mean_tpot", "mean_tpot"), ("goodput", "goodput"), ("span", "span_s"))


def _digest(name):
    path = H.GOLDEN / f"digest_{name}.npz"
    if not path.exists():
        pytest.skip(f"{path.name} not generated")
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


def check_against_digest(summaries, d):
    st = summaries["status"].astype(np.int64)
    np.testing.assert_array_equal(st, d["status"], err_msg="status (ok / stalled)")
    ok = d["status"] == 0
    H.assert_same_f64(summaries["stall_time"][~ok], d["stall_time"][~ok], "stall time")
    np.testing.assert_array_equal(summaries["decision_hash"][ok], d["decision_hash"][ok], err_msg="decision digest")
    np.testing.assert_array_equal(summaries["n_decisions"][ok], d["n_decisions"][ok], err_msg="n_decisions")
    np.testing.assert_array_equal(summaries["n_flips"][ok], d["n_flips"][ok], err_msg="n_flips")
    for f, g in DIGEST_FIELDS:
        H.assert_same_f64(summaries[f][ok], d[g][ok], f)


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_whole_sweep_matches_reference_digest(evaluator, name):
    d = _digest(name)
    scs = getattr(W, name)(d["id"])
    cb = compile_batch(scs, engine.STALL_EVENT_LIMIT)
    got = evaluator.execute(cb, OutputSpec(), dispatch_order(cb))
    check_against_digest(got.summaries, d)
