"""Shared test plumbing: golden fixtures, the CPU oracle, the host SIMT
emulator of the kernel, and field-by-field comparison helpers.

The oracle (oracle/build/libpdsim_oracle.so) and the emulator
(build/libarrow_emu.so) are test infrastructure only; the product package
never loads them.
"""

from __future__ import annotations

import ctypes
import json
import math
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_2505_11916_b200 import _abi  # noqa: E402
from paper_2505_11916_b200._buffers import HostBuffers, OutputSpec  # noqa: E402
from paper_2505_11916_b200._compile import Scenario, TraceEntry, compile_batch  # noqa: E402
from paper_2505_11916_b200.config import config_from_values  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"

_libs: dict = {}


def _build(target: str) -> None:
    """Incremental build under a file lock: pytest-xdist workers must not
    rebuild (and dlopen) the same library concurrently."""
    import fcntl

    (ROOT / "build").mkdir(exist_ok=True)
    with open(ROOT / "build" / ".build.lock", "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        subprocess.run(["make", "-s", "-j8", "-C", str(ROOT), target], check=True)


def oracle_lib() -> ctypes.CDLL:
    if "oracle" not in _libs:
        path = ROOT / "oracle" / "build" / "libpdsim_oracle.so"
        _build("oracle")          # incremental: rebuilds when the shared header changed
        lib = ctypes.CDLL(str(path))
        lib.pdsim_oracle_run_batch.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.pdsim_oracle_run_batch.restype = ctypes.c_int
        lib.pdsim_oracle_run_batch_timed.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        lib.pdsim_oracle_run_batch_timed.restype = ctypes.c_int
        lib.pdsim_oracle_pysum.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        lib.pdsim_oracle_pysum.restype = ctypes.c_double
        lib.pdsim_oracle_decision_hash.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        lib.pdsim_oracle_decision_hash.restype = ctypes.c_uint64
        _libs["oracle"] = lib
    return _libs["oracle"]


def emu_lib(variant: str = "") -> ctypes.CDLL:
    """variant "" is the kernel source as shipped; "wide" widens the delay
    intervals so that most dispatch decisions take the exact-fold fallback;
    "mut" carries test-only mutants selected per call (run_emu(mutant=...)):
    "tie" merges equal-time burst finals in reversed order, "kv" mis-reserves
    migration KV (the audit checks are compiled in); "audit" is the shipped
    source with the per-step audit checks."""
    key = "emu" + variant
    if key not in _libs:
        path = ROOT / "build" / {"": "libarrow_emu.so", "wide": "libarrow_emu_wide.so",
                                 "mut": "libarrow_emu_mut.so", "audit": "libarrow_emu_audit.so"}[variant]
        _build("emu")
        lib = ctypes.CDLL(str(path))
        lib.arrow_emu_run.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.arrow_emu_run.restype = ctypes.c_int
        _libs[key] = lib
    return _libs[key]


def golden_index() -> list[dict]:
    return json.loads((GOLDEN / "index.json").read_text())["scenarios"]


def golden_arrays(meta: dict) -> dict:
    with np.load(GOLDEN / meta["file"]) as z:
        return {k: z[k] for k in z.files}


def golden_scenario(meta: dict, arrays: dict, **overrides) -> Scenario:
    values = dict(meta["values"])
    values.update(overrides)
    cfg = config_from_values(values)
    entry = TraceEntry(arrays["arrival"], arrays["input_len"], arrays["output_len"], arrays["ids"])
    return Scenario(entry, cfg, meta["scale"], meta["name"])


def compile_golden(metas_arrays, validate=True):
    scs = [golden_scenario(m, a) for m, a in metas_arrays]
    limits = {m["stall_limit"] for m, _ in metas_arrays}
    assert len(limits) == 1
    return compile_batch(scs, limits.pop(), validate=validate)


FULL = OutputSpec(requests=True, decisions=True, snapshots=True, iterlog=True, diag=True)


def spec_for(metas_arrays, base: OutputSpec = FULL) -> OutputSpec:
    """``base`` with a decision-log capacity large enough for every fixture in
    the group (Arrow on the C3 code-like trace logs ~2 500 flips, beyond the
    default 2n + 64 entries)."""
    factor = 1.0
    for m, a in metas_arrays:
        if "decisions" in a:
            factor = max(factor, (len(a["decisions"]) + 64) / (2 * len(a["arrival"]) + 64))
    return OutputSpec(**{**base.__dict__, "decision_factor": math.ceil(factor * 8) / 8})


def run_oracle(cb, spec=FULL, threads=1, tokens=False) -> HostBuffers:
    spec = OutputSpec(**{**spec.__dict__, "tokens": tokens})
    hb = HostBuffers(cb, spec)
    b = hb.host_struct()
    oracle_lib().pdsim_oracle_run_batch(ctypes.addressof(b), threads)
    return hb


def run_oracle_timed(cb, threads=0):
    """Summaries of the CPU port plus each scenario's wall seconds on its
    worker thread (bench.py's CPU baseline)."""
    hb = HostBuffers(cb, OutputSpec())
    b = hb.host_struct()
    secs = np.zeros(cb.n, dtype=np.float64)
    used = oracle_lib().pdsim_oracle_run_batch_timed(ctypes.addressof(b), threads, secs.ctypes.data)
    return hb, secs, used


def run_emu(cb, spec=FULL, width=8, variant: str = "", mutant: str | None = None) -> HostBuffers:
    """mutant (variant "mut" only): ARROW_MUTANT=tie|kv for this call."""
    import os

    hb = HostBuffers(cb, spec)
    b = hb.host_struct()
    if mutant:
        assert variant == "mut"
        os.environ["ARROW_MUTANT"] = mutant
    try:
        rc = emu_lib(variant).arrow_emu_run(ctypes.addressof(b), width)
    finally:
        os.environ.pop("ARROW_MUTANT", None)
    assert rc == 0, rc
    return hb


def bits(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float64).view(np.uint64)


def assert_same_f64(a, b, what):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, f"{what}: shape {a.shape} vs {b.shape}"
    same = (bits(a) == bits(b)) | (np.isnan(a) & np.isnan(b))
    if not same.all():
        i = int(np.argmin(same))
        raise AssertionError(f"{what}: first mismatch at {i}: {a[i]!r} vs {b[i]!r} ({int((~same).sum())} total)")


def assert_same_decisions(got: np.ndarray, exp: np.ndarray, what="decisions"):
    n = min(len(got), len(exp))
    for k in range(n):
        g, e = got[k], exp[k]
        if (
            bits(g["time"]) != bits(e["time"])
            or int(g["request"]) != int(e["request"])
            or int(g["instance"]) != int(e["instance"])
            or int(g["kind"]) != int(e["kind"])
            or int(g["code"]) != int(e["code"])
        ):
            raise AssertionError(f"{what}: first divergence at #{k}: got {describe(g)} expected {describe(e)}")
    assert len(got) == len(exp), f"{what}: {len(got)} entries vs {len(exp)} expected"


def describe(d) -> str:
    kind = int(d["kind"])
    if kind == 2:
        code = int(d["code"])
        return (f"flip t={float(d['time'])!r} inst={int(d['instance'])} {_abi.POOL_NAMES[(code >> 3) & 3]}->"
                f"{_abi.POOL_NAMES[(code >> 5) & 3]} {_abi.TRIGGER_NAMES[code & 7]}")
    return (f"{_abi.DECISION_KIND_NAMES[kind]} t={float(d['time'])!r} req={int(d['request'])} "
            f"inst={int(d['instance'])} {_abi.BRANCH_NAMES[int(d['code'])]}")


SUMMARY_KEYS = ("attainment", "p90_ttft", "p90_tpot", "mean_ttft", "mean_tpot", "goodput", "span_s")


def check_vs_golden(meta: dict, arrays: dict, hb: HostBuffers, s: int = 0, snapshots=True) -> None:
    """Bitwise comparison of one scenario's outputs with the reference's."""
    summ = hb.summaries[s]
    err = meta["error"]
    if err is not None and err[0] == "SimulationStallError":
        assert summ["status"] == _abi.STALLED, f"status {_abi.STATUS_NAMES[summ['status']]}, expected stall"
        t = float(err[1].split("t=", 1)[1].split(":", 1)[0])
        assert bits(summ["stall_time"]) == bits(t), (summ["stall_time"], t)
        return
    assert err is None, err
    assert summ["status"] == _abi.OK, f"status {_abi.STATUS_NAMES[summ['status']]} overflow {summ['overflow']}"
    assert_same_decisions(hb.decisions_of(s), arrays["decisions"])
    sl = hb.req_slice(s)
    assert_same_f64(hb.req_first[sl], arrays["first"], "first token")
    assert_same_f64(hb.req_last[sl], arrays["last"], "last token")
    exp = meta["summary"]
    for k in SUMMARY_KEYS:
        got = float(summ["span" if k == "span_s" else k])
        assert bits(got) == bits(exp[k]) or (math.isinf(got) and math.isinf(exp[k])), (k, got, exp[k])
    assert int(summ["n_ok"]) == int(((arrays["flags"] >> 2) & 1).sum())
    assert int(summ["n_flips"]) == len(arrays["transitions"])
    if snapshots and "snapshots" in arrays and hb.snapshots is not None:
        got = hb.snapshots_of(s)
        exp_s = arrays["snapshots"]
        assert len(got) == len(exp_s), ("snapshots", len(got), len(exp_s))
        for f in ("instance", "pool", "running_tokens", "kv_used", "queue_len", "prefill_count", "decode_count"):
            np.testing.assert_array_equal(got[f], exp_s[f], err_msg=f"snapshot {f}")
        for f in ("time", "pred_delay", "avg_interval"):
            assert_same_f64(got[f], exp_s[f], f"snapshot {f}")


def golden_free_decisions(hb: HostBuffers, s: int, cb) -> list[dict]:
    """Decision dicts (reference format) from raw oracle outputs."""
    from paper_2505_11916_b200 import _results

    return _results.decision_dicts(hb, s, cb.table.entries[cb.trace_index[s]].ids)


def lockstep_scenarios():
    """Groups of identical requests arriving at the same instant on eight
    identical instances: dispatch, batches and iteration times coincide
    across instances, so many events share exact times and the (time, kind,
    seq) tie-breaks decide the order.  One scenario per policy."""
    from paper_2505_11916_b200 import workloads as W
    from paper_2505_11916_b200._compile import Scenario
    from paper_2505_11916_b200.core import TraceRequest

    trace = []
    for g in range(12):
        for j in range(8):
            trace.append(TraceRequest(len(trace), 0.25 * g, 64 + 32 * (g % 3), 24 + 8 * (g % 2)))
    base = W.sweep_base(8)
    return [Scenario(trace, W.policy_config(base, p, 8), 1.0, p) for p in W.POLICIES]


def assert_same_run(got, exp, n: int) -> None:
    """Every summary field, per-request time and dispatch target equal."""
    from paper_2505_11916_b200 import _abi

    for s in range(n):
        g, e = got.summaries[s], exp.summaries[s]
        for f in ("status", "n_completed", "n_ok", "n_flips", "n_events", "n_iterations", "n_decisions",
                  "n_ticks", "decision_hash"):
            assert int(g[f]) == int(e[f]), (s, f, g[f], e[f])
        for f in ("stall_time", "attainment", "p90_ttft", "p90_tpot", "mean_ttft", "mean_tpot", "goodput", "span"):
            assert_same_f64([g[f]], [e[f]], f"scenario {s} {f}")
    assert_same_f64(got.req_first, exp.req_first, "first")
    for s in range(n):
        if int(exp.summaries[s]["status"]) == _abi.OK:
            sl = got.req_slice(s)
            assert_same_f64(got.req_last[sl], exp.req_last[sl], f"scenario {s} last")
    np.testing.assert_array_equal(got.req_prefill, exp.req_prefill)
    np.testing.assert_array_equal(got.req_decode, exp.req_decode)


class OracleEvaluator:
    """The CPU oracle behind the CudaEvaluator interface (.execute), so tests
    can drive the package's host-side paths (result assembly, writers, CLI)
    on a machine without a GPU.  Test-only: the product has no CPU path."""

    def execute(self, cb, spec, order=None):
        return run_oracle(cb, spec)


def use_oracle_backend(monkeypatch) -> None:
    from paper_2505_11916_b200 import _backend

    ev = OracleEvaluator()
    monkeypatch.setattr(_backend, "default_evaluator", lambda audit=False: ev)
