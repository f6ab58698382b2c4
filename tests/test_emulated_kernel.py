"""The CUDA kernel's scheduling logic (csrc/sim_core.cuh), compiled for the
host and run by a thread-per-lane warp emulator, against the reference's
golden outputs.  This is how the kernel is checked in a container without a
GPU; the `gpu` tests repeat the comparison on the B200."""

from __future__ import annotations

import pytest

import harness as H

INDEX = H.golden_index()
SMALL = [
    m
    for m in INDEX
    if not (m["error"] and m["error"][0] == "ValueError") and not m["name"].startswith(("c2_", "c3_", "c4_", "c5_"))
]
# BASELINE C3 / C5 fixtures through the emulator: one per (trace, policy) of
# C3 and the C5 ids with N <= 8 (the thread-per-lane emulator is slow for
# wide clusters; every C3/C4/C5 fixture runs on the B200 in test_gpu_parity).
R2 = [m for m in INDEX if m["name"] in (
    "c3_code_arrow_0", "c3_code_static-pd_1", "c3_code_colocated_2", "c3_chat_arrow_3", "c3_chat_static-pd_4",
    "c3_chat_colocated_5")] + [m for m in INDEX if m["name"].startswith("c5_") and m["values"]["instances"] <= 8]


@pytest.mark.parametrize("meta", SMALL, ids=[m["name"] for m in SMALL])
def test_emulated_kernel_matches_reference(meta):
    arrays = H.golden_arrays(meta)
    cb = H.compile_golden([(meta, arrays)])
    hb = H.run_emu(cb, width=8)
    H.check_vs_golden(meta, arrays, hb)


@pytest.mark.parametrize("meta", R2, ids=[m["name"] for m in R2])
def test_emulated_kernel_matches_reference_baseline_configs(meta):
    arrays = H.golden_arrays(meta)
    cb = H.compile_golden([(meta, arrays)])
    hb = H.run_emu(cb, H.spec_for([(meta, arrays)]), width=8)
    H.check_vs_golden(meta, arrays, hb)


def test_emulated_kernel_two_slots_per_lane():
    """Instances i and i+W share a lane (IPL=2 register slots): 12 instances
    on a 4-lane emulated warp."""
    meta = next(m for m in INDEX if m["name"] == "determinism_600")
    arrays = H.golden_arrays(meta)
    cb = H.compile_golden([(meta, arrays)])
    hb = H.run_emu(cb, width=4)
    H.check_vs_golden(meta, arrays, hb)


def test_emulated_kernel_batch_of_scenarios():
    """Several scenarios through one (emulated) slot, back to back: state
    from one scenario must not leak into the next."""
    names = ["small_arrow_2_2", "rr_small", "conservation_slo", "overload_flips", "fuzz_05"]
    items = [(m, H.golden_arrays(m)) for m in INDEX if m["name"] in names]
    groups: dict = {}
    for m, a in items:
        groups.setdefault(m["stall_limit"], []).append((m, a))
    for group in groups.values():
        cb = H.compile_golden(group)
        hb = H.run_emu(cb, width=8)
        for s, (m, a) in enumerate(group):
            H.check_vs_golden(m, a, hb, s)


@pytest.mark.parametrize("index", [9, 27, 41, 52, 84])
def test_emulated_kernel_matches_oracle_on_c2_points(index):
    """C2 sweep points under heavy KV pressure (queued migrations, waiting
    decodes, flips) — where chain bursts must stop before loud events —
    against the CPU oracle: every summary field and per-request time."""
    from paper_2505_11916_b200 import workloads as W
    from paper_2505_11916_b200._buffers import OutputSpec
    from paper_2505_11916_b200._compile import compile_batch

    cb = compile_batch([W.c2()[index]], 500_000)
    spec = OutputSpec(requests=True, decisions=True)
    got = H.run_emu(cb, spec, width=8)
    exp = H.run_oracle(cb, spec)
    g, e = got.summaries[0], exp.summaries[0]
    for f in ("status", "n_completed", "n_ok", "n_flips", "n_events", "n_iterations", "n_decisions", "decision_hash"):
        assert int(g[f]) == int(e[f]), f
    H.assert_same_f64(got.req_first, exp.req_first, "first")
    H.assert_same_f64([g["stall_time"]], [e["stall_time"]], "stall time")
    if int(e["status"]) == 0:       # a stalled run raises; its partial records are never observed
        H.assert_same_f64(got.req_last, exp.req_last, "last")
        H.assert_same_decisions(got.decisions_of(0), exp.decisions_of(0))


WIDE = [m for m in SMALL if m["name"].startswith(("fuzz_", "overload", "c1_", "small_", "migration", "tight", "adv_delay"))]


@pytest.mark.parametrize("meta", WIDE, ids=[m["name"] for m in WIDE])
def test_exact_fold_fallbacks_match_reference(meta):
    """Dispatches decide from delay intervals and fold exactly only when the
    interval cannot settle them; with intervals 2^40 times wider (most
    decisions then take the exact fallbacks) the kernel source must still
    reproduce the reference bit for bit."""
    arrays = H.golden_arrays(meta)
    cb = H.compile_golden([(meta, arrays)])
    hb = H.run_emu(cb, width=8, variant="wide")
    H.check_vs_golden(meta, arrays, hb)


NO_ITERLOG = H.OutputSpec(requests=True, decisions=True, snapshots=True, diag=True)


@pytest.mark.parametrize("meta", SMALL, ids=[m["name"] for m in SMALL])
def test_emulated_kernel_without_iteration_log(meta):
    """Without the per-iteration log output (the sweep configuration), chain
    bursts take their steady-stretch fast path; decisions, token times,
    summaries and snapshots must not change."""
    arrays = H.golden_arrays(meta)
    cb = H.compile_golden([(meta, arrays)])
    hb = H.run_emu(cb, NO_ITERLOG, width=8)
    H.check_vs_golden(meta, arrays, hb)


def test_emulated_kernel_lockstep_instances_match_oracle():
    """Simultaneous identical requests on identical instances: exact ties
    between event times (tests/harness.py: lockstep_scenarios)."""
    from paper_2505_11916_b200._buffers import OutputSpec
    from paper_2505_11916_b200._compile import compile_batch

    cb = compile_batch(H.lockstep_scenarios(), 500_000)
    spec = OutputSpec(requests=True)
    got = H.run_emu(cb, spec, width=8)
    exp = H.run_oracle(cb, spec)
    H.assert_same_run(got, exp, cb.n)
    assert (exp.summaries["status"] == 0).all()


def test_emulated_kernel_adversarial_predictors_match_oracle():
    """Mixed-sign, cancelling predictor terms (heavy profiling noise) through
    the kernel source, shipped and wide-interval builds, against the oracle."""
    from test_gpu_sweeps import _adversarial_predictor_scenarios, _compare
    from paper_2505_11916_b200._buffers import OutputSpec
    from paper_2505_11916_b200._compile import compile_batch

    cb = compile_batch(_adversarial_predictor_scenarios(12, 12), 20000)
    spec = OutputSpec(requests=True)
    exp = H.run_oracle(cb, spec, threads=0)
    for variant in ("", "wide"):
        _compare(H.run_emu(cb, spec, width=8, variant=variant), exp, cb.n)
