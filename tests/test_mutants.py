"""The tests have teeth: test-only mutants of the kernel source (host
emulator build with -DARROW_MUTANTS, selected per call) must be caught.

* "tie": the chain-burst merge assigns equal-time final pushes in reversed
  order.  The tie_lockstep_* fixtures (written by the real reference,
  oracle/scenarios.py:tie_lockstep_trace) make that order visible in the
  decision stream; the shipped source reproduces them, the mutant does not.
* "kv": a migration reserves one KV token too many.  The audit build's
  per-step checks (RunConfig.audit, engine.py:279-282) end the run with
  ARROW_AUDIT_FAILED, which the shim raises as AssertionError; the shipped
  source passes the same checks on every golden scenario.
"""

from __future__ import annotations

import pytest

import harness as H
from paper_2505_11916_b200 import _abi

INDEX = {m["name"]: m for m in H.golden_index()}
TIES = sorted(n for n in INDEX if n.startswith("tie_lockstep_"))


def _load(name):
    m = INDEX[name]
    a = H.golden_arrays(m)
    return m, a, H.compile_golden([(m, a)])


def test_tie_fixtures_reach_the_merge_fallback_observably():
    assert len(TIES) >= 3
    caught = 0
    for name in TIES:
        m, a, cb = _load(name)
        H.check_vs_golden(m, a, H.run_emu(cb, width=8))               # shipped source: exact
        H.check_vs_golden(m, a, H.run_emu(cb, width=8, variant="mut"))  # mutant build, mutant off
        try:
            H.check_vs_golden(m, a, H.run_emu(cb, width=8, variant="mut", mutant="tie"))
        except AssertionError as e:
            assert "decisions" in str(e)
            caught += 1
    assert caught >= 3, f"the reversed tie merge was caught on only {caught} of {len(TIES)} fixtures"


@pytest.mark.parametrize("name", ["small_arrow_2_2", "conservation_slo", "migration_gap", "c1_rate4"])
def test_audit_catches_kv_mutant(name):
    m, a, cb = _load(name)
    spec = H.spec_for([(m, a)])
    assert int(H.run_emu(cb, spec, width=8, variant="audit").summaries[0]["status"]) == _abi.OK
    hb = H.run_emu(cb, spec, width=8, variant="mut", mutant="kv")
    assert int(hb.summaries[0]["status"]) == _abi.AUDIT_FAILED
    from paper_2505_11916_b200 import _results

    with pytest.raises(AssertionError, match="audit"):
        _results.raise_for_status(hb, 0)


AUDITED = [n for n, m in INDEX.items() if not (m["error"] and m["error"][0] == "ValueError")
           and not n.startswith(("c2_", "c3_", "c4_", "c5_"))]


@pytest.mark.parametrize("name", AUDITED[::3])
def test_audit_build_passes_golden(name):
    """Every third small golden scenario through the audit build on CPU (all
    of them, plus C2-C5, run through the audit build on the B200)."""
    m, a, cb = _load(name)
    H.check_vs_golden(m, a, H.run_emu(cb, H.spec_for([(m, a)]), width=8, variant="audit"))


@pytest.mark.gpu
def test_audit_build_on_gpu_golden():
    """RunConfig.audit=True selects libarrow_sim_audit.so; every golden
    scenario passes its per-step checks on the B200."""
    from paper_2505_11916_b200._backend import CudaEvaluator

    ev = CudaEvaluator(audit=True)
    items = [(m, H.golden_arrays(m)) for m in INDEX.values() if not (m["error"] and m["error"][0] == "ValueError")]
    by_limit: dict = {}
    for m, a in items:
        by_limit.setdefault(m["stall_limit"], []).append((m, a))
    for group in by_limit.values():
        cb = H.compile_golden(group)
        hb = ev.execute(cb, H.spec_for(group))
        for s, (m, a) in enumerate(group):
            H.check_vs_golden(m, a, hb, s)


@pytest.mark.gpu
def test_run_with_audit_config_uses_audit_build():
    import dataclasses

    import paper_2505_11916_b200 as arrow
    from paper_2505_11916_b200 import _backend

    m = INDEX["small_arrow_2_2"]
    a = H.golden_arrays(m)
    sc = H.golden_scenario(m, a)
    cfg = dataclasses.replace(sc.config, audit=True)
    trace = [arrow.TraceRequest(int(i), float(t), int(x), int(y))
             for i, t, x, y in zip(a["ids"], a["arrival"], a["input_len"], a["output_len"])]
    res = arrow.run(trace, cfg)
    assert [r.token_times[0] for r in res.records] == a["first"].tolist()
    assert any(getattr(ev, "audit", False) for ev in _backend._default.values())
