"""Pin the CPU oracle (and the host-side numpy pieces) to the real
reference's outputs stored in tests/golden/ (oracle/gen_golden.py)."""

from __future__ import annotations

import ctypes
import math

import numpy as np
import pytest

import harness as H
from paper_2505_11916_b200 import cost_model, traces
from paper_2505_11916_b200._compile import resolve_max_tokens, resolve_predictor
from paper_2505_11916_b200.config import config_from_values

INDEX = H.golden_index()
RUNNABLE = [m for m in INDEX if not (m["error"] and m["error"][0] == "ValueError")]
INVALID = [m for m in INDEX if m["error"] and m["error"][0] == "ValueError"]


@pytest.mark.parametrize("meta", RUNNABLE, ids=[m["name"] for m in RUNNABLE])
def test_oracle_matches_reference(meta):
    arrays = H.golden_arrays(meta)
    cb = H.compile_golden([(meta, arrays)])
    hb = H.run_oracle(cb, H.spec_for([(meta, arrays)]), tokens=bool(meta["full"]))
    H.check_vs_golden(meta, arrays, hb)
    if meta["full"] and meta["error"] is None:
        got = np.concatenate([hb.tokens_of(0, r) for r in range(len(arrays["arrival"]))])
        H.assert_same_f64(got, arrays["token_times"], "token times")


@pytest.mark.parametrize("meta", INVALID, ids=[m["name"] for m in INVALID])
def test_validation_errors_match_reference(meta):
    arrays = H.golden_arrays(meta)
    with pytest.raises(ValueError) as exc:
        H.compile_golden([(meta, arrays)])
    assert str(exc.value) == meta["error"][1]


@pytest.mark.parametrize("meta", RUNNABLE[:20], ids=[m["name"] for m in RUNNABLE[:20]])
def test_host_resolution_matches_reference(meta):
    """Predictor fit (numpy lstsq) and token cap resolved like engine.py:128-134."""
    arrays = H.golden_arrays(meta)
    cfg = config_from_values(meta["values"])
    p = resolve_predictor(cfg)
    H.assert_same_f64([p.a2, p.a1, p.a0], arrays["predictor"], "predictor")
    assert resolve_max_tokens(cfg) == int(arrays["max_tokens"][0])


@pytest.fixture(scope="module")
def kav():
    with np.load(H.GOLDEN / "known_answers.npz") as z:
        return {k: z[k] for k in z.files}


def _as_rows(trace):
    return np.array([(r.arrival, r.input_len, r.output_len) for r in trace])


def test_generators_match_reference(kav):
    p0 = traces.SyntheticParams(50.0, 3.0, math.log(300), 0.5, math.log(60), 0.4, seed=11)
    p1 = traces.SyntheticParams(30.0, 2.0, math.log(1500), 0.9, math.log(40), 0.8,
                                bursts=(traces.BurstEpisode(5.0, 5.0, 5.0),), max_input=8000, max_output=1000,
                                seed=101)
    H.assert_same_f64(_as_rows(traces.gen_synthetic(p0)), kav["synthetic_0"], "synthetic 0")
    H.assert_same_f64(_as_rows(traces.gen_synthetic(p1)), kav["synthetic_1"], "synthetic 1")
    H.assert_same_f64(_as_rows(traces.bundled_bursty_trace()), kav["bursty"], "bursty")
    H.assert_same_f64(_as_rows(traces.bundled_ramp_trace()), kav["ramp"], "ramp")


def test_fits_match_reference(kav):
    for seed, noise, a2, a1, a0, f2, f1, f0 in kav["fits"]:
        rng = np.random.default_rng(int(seed))
        grid = cost_model.default_profile_grid(16384, 16)
        samples = cost_model.profile_prefill(cost_model.PrefillCostParams(a2, a1, a0), grid, float(noise), rng)
        f = cost_model.fit_quadratic(samples)
        H.assert_same_f64([f.a2, f.a1, f.a0], [f2, f1, f0], f"fit seed={seed} noise={noise}")


def test_token_cap_matches_reference(kav):
    got = [
        cost_model.max_running_tokens(cost_model.DecodeCostParams(2e-5, 5e-3), 16000, 0.1),
        cost_model.max_running_tokens(cost_model.DecodeCostParams(1e-4, 4e-3), 3000, 0.1),
        cost_model.max_running_tokens(cost_model.DecodeCostParams(2e-5, 5e-3), 16000, 0.025),
    ]
    assert got == kav["max_tokens"].tolist()


def test_oracle_pysum_is_cpython_sum(kav):
    """The compensated float sum the device reproduces (CPython 3.12
    builtin sum) against the interpreter's own results."""
    lib = H.oracle_lib()
    vals = np.ascontiguousarray(kav["pysum_values"])
    off = 0
    for n, exp in zip(kav["pysum_lengths"], kav["pysum_results"]):
        seg = np.ascontiguousarray(vals[off : off + n])
        got = lib.pdsim_oracle_pysum(seg.ctypes.data, int(n))
        H.assert_same_f64([got], [exp], f"sum of {n}")
        H.assert_same_f64([got], [sum(seg.tolist())], "interpreter sum")
        off += n


def test_decision_hash_definition():
    """The FNV digest the kernel and oracle compute equals the Python one."""
    meta = next(m for m in RUNNABLE if m["name"] == "c1_rate4")
    arrays = H.golden_arrays(meta)
    cb = H.compile_golden([(meta, arrays)])
    hb = H.run_oracle(cb)
    from paper_2505_11916_b200._abi import fnv_decision_hash

    dec = np.ascontiguousarray(hb.decisions_of(0))
    assert fnv_decision_hash(dec) == int(hb.summaries[0]["decision_hash"])
    lib = H.oracle_lib()
    assert lib.pdsim_oracle_decision_hash(dec.ctypes.data, len(dec)) == int(hb.summaries[0]["decision_hash"])


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_oracle_matches_reference_digest_sample(name):
    """Every 16th scenario of the whole-sweep reference digests through the
    CPU oracle (the B200 runs all of them: test_gpu_sweeps.py)."""
    from paper_2505_11916_b200 import engine
    from paper_2505_11916_b200 import workloads as W
    from paper_2505_11916_b200._buffers import OutputSpec
    from paper_2505_11916_b200._compile import compile_batch

    import test_gpu_sweeps as T

    d = T._digest(name)
    sel = np.arange(0, len(d["id"]), 16)
    d = {k: v[sel] for k, v in d.items()}
    cb = compile_batch(getattr(W, name)(d["id"]), engine.STALL_EVENT_LIMIT)
    T.check_against_digest(H.run_oracle(cb, OutputSpec(), threads=0).summaries, d)
