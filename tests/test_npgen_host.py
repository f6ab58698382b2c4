"""Device workload generator, checked WITHOUT a GPU.

The generator source (csrc/npgen.cuh) is compiled for the host
(build/libnpgen_host.so, test-only) and compared bit for bit with:
  * numpy itself: SeedSequence/PCG64 states, raw / random / exponential /
    normal streams (the reference's RNG dependency, traces.py:161-173);
  * the image's libm: glibc exp and log1p, which numpy's ziggurats and
    Python's math.exp call;
  * the real reference's gen_synthetic on the golden catalogue
    (tests/golden/synth_traces.npz) and this repo's numpy host generator on
    seeded random parameter sets;
and the committed table header is checked against the installed numpy.
"""

from __future__ import annotations

import ctypes
import subprocess
import sys

import numpy as np
import pytest

import harness as H
import synth_harness as SH
from paper_2505_11916_b200 import _abi
from paper_2505_11916_b200.device_traces import expected_requests, seed_words, synth_record


def test_table_header_matches_installed_numpy(tmp_path):
    out = tmp_path / "t.h"
    subprocess.run([sys.executable, str(H.ROOT / "scripts" / "gen_npgen_tables.py"), str(out)], check=True,
                   capture_output=True)
    committed = (H.ROOT / "paper_2505_11916_b200" / "csrc" / "npgen_tables.h").read_text()
    fresh = out.read_text()
    strip = lambda s: "\n".join(l for l in s.splitlines() if "numpy" not in l)  # noqa: E731  version line
    assert strip(committed) == strip(fresh)


@pytest.mark.parametrize("kind,n", [(0, 3_000_000), (1, 1_000_000), (2, 1_000_000), (3, 1_000_000), (4, 3_000_000)])
def test_libm_emulation_bit_exact(kind, n):
    lib = SH.npgen_lib()
    bad_x = ctypes.c_double(0.0)
    bad = lib.npgen_check_libm(kind, n, 0x9E3779B97F4A7C15 + kind, ctypes.byref(bad_x))
    assert bad == 0, f"{bad} mismatches vs libm, first at x={bad_x.value!r}"


def test_libm_special_values():
    lib = SH.npgen_lib()
    libm = ctypes.CDLL("libm.so.6")
    libm.log1p.argtypes = libm.exp.argtypes = [ctypes.c_double]
    libm.log1p.restype = libm.exp.restype = ctypes.c_double
    xs = [0.0, -0.0, 1e-300, -1e-300, 2**-54, -(2**-54), 2**-29, -(2**-29), -0.2928, -0.2929, 0.41421, 0.41423,
          -1.0 + 2**-52, 1.0, 2.0, 2**53, 2**60, 1e300, float("inf"), -1.0, -2.0]
    for x in xs:
        a, b = lib.npgen_log1p(x), libm.log1p(x)
        assert SH.isclose_bits(a, b), ("log1p", x, a, b)
    for x in [0.0, -0.0, 1e-20, -1e-20, 2**-54, 709.0, 709.78, 710.0, -708.0, -740.0, -745.1, -800.0, 1000.0,
              float("inf"), float("-inf"), 511.9, 512.0, -512.0, 1.5, -1.5]:
        a, b = lib.npgen_exp(x), libm.exp(x)
        assert SH.isclose_bits(a, b), ("exp", x, a, b)


@pytest.mark.parametrize("seed", [0, 1, 2, 7, 42, 20240817, 2**32 - 1, 2**32, 2**40 + 5, 2**64 + 3, 2**100 + 12345,
                                  2**255 - 19])
def test_seed_sequence_pcg64_state(seed):
    lib = SH.npgen_lib()
    w = seed_words(seed)
    arr = (ctypes.c_uint32 * len(w))(*w)
    out = (ctypes.c_uint64 * 4)()
    lib.npgen_seed_state(arr, len(w), out)
    assert list(out) == SH.seed_state_words(seed)


def test_seed_words_validation():
    with pytest.raises(ValueError, match="non-negative"):
        seed_words(-1)
    with pytest.raises(TypeError):
        seed_words(1.5)
    assert len(seed_words(None)) >= 1


@pytest.mark.parametrize("seed", [0, 5, 20240817, 2**70 + 1])
def test_streams_bit_exact(seed):
    lib = SH.npgen_lib()
    n = 400_000
    for kind, ref in (
        (0, lambda: np.random.PCG64(seed).random_raw(n)),
        (1, lambda: np.random.default_rng(seed).random(n)),
        (2, lambda: np.random.default_rng(seed).standard_exponential(n)),
        (3, lambda: np.random.default_rng(seed).standard_normal(n)),
    ):
        st = (ctypes.c_uint64 * 4)(*SH.seed_state_words(seed))
        out = np.zeros(n, dtype=np.uint64 if kind == 0 else np.float64)
        lib.npgen_draw(st, kind, n, out.ctypes.data)
        exp = ref()
        assert np.array_equal(out.view(np.uint64), np.asarray(exp).view(np.uint64)), kind


def test_golden_catalogue_host_emulation():
    entries = SH.golden_entries()
    got, res = SH.host_emulated_batch([p for _, p, _ in entries])
    for (name, _p, exp), g, r in zip(entries, got, res):
        SH.assert_trace_equal(name, g, exp)
        if len(exp[0]):
            assert SH.isclose_bits(float(r["first_arrival"]), float(exp[0][0]))
            assert SH.isclose_bits(float(r["last_arrival"]), float(exp[0][-1]))
            assert int(r["max_kv"]) == int((exp[1] + exp[2]).max())
            assert int(r["sum_output"]) == int(exp[2].sum())


def test_random_params_host_emulation():
    rng = np.random.default_rng(2505)
    params = [SH.random_params(rng) for _ in range(40)]
    got, _ = SH.host_emulated_batch(params)
    for k, (p, g) in enumerate(zip(params, got)):
        SH.assert_trace_equal(f"random[{k}] {p}", g, SH.host_trace_arrays(p))


def test_capacity_estimate_covers_catalogue():
    for name, p, exp in SH.golden_entries():
        lam = expected_requests(p)
        assert len(exp[0]) <= lam + 10 * lam**0.5 + 32, name


def test_synth_record_limits():
    p = SH.params_of(dict(duration_s=1.0, base_rate=1.0, input_log_mean=1.0, input_log_sigma=0.1,
                          output_log_mean=1.0, output_log_sigma=0.1))
    from dataclasses import replace

    with pytest.raises(ValueError, match="finite"):
        synth_record(replace(p, duration_s=float("inf")), 0, 1)
    with pytest.raises(ValueError, match="2\\*\\*31"):
        synth_record(replace(p, max_input=2**31), 0, 1)
    rec = synth_record(replace(p, seed=2**40 + 7), 5, 9)
    assert rec["n_seed_words"] == 2 and rec["out_offset"] == 5 and rec["capacity"] == 9
    assert _abi.SYNTH_DTYPE.itemsize == rec.nbytes


def _fake_set(traces):
    """A DeviceTraceSet over CPU tensors (host-emulated generation), to test
    the scenario compiler's device-trace path without a GPU."""
    import torch

    from paper_2505_11916_b200.device_traces import DeviceTraceSet

    params = [SH.params_of(kw) for _, kw in traces]
    got, res = SH.host_emulated_batch(params)
    offs = np.cumsum([0] + [len(g[0]) for g in got])[:-1].astype(np.int64)
    arr = torch.from_numpy(np.concatenate([g[0] for g in got]))
    inp = torch.from_numpy(np.concatenate([g[1] for g in got]).astype(np.int32))
    out = torch.from_numpy(np.concatenate([g[2] for g in got]).astype(np.int32))
    return DeviceTraceSet(params, arr, inp, out, offs, res, torch.device("cpu")), got


def test_compile_batch_with_device_traces():
    import paper_2505_11916_b200 as arrow
    from paper_2505_11916_b200._compile import Scenario, compile_batch, dispatch_order

    cat = dict(SH.catalogue())
    ts, got = _fake_set([("a", dict(cat["small"], seed=1)), ("b", dict(cat["small"], seed=2))])
    import scenarios as S

    cfg = arrow.config_from_values(S.cfg(instances=4, kv_capacity_tokens=16000))
    cb = compile_batch([Scenario(ts[1], cfg, 0.5), Scenario(ts[0], cfg, 1.0), Scenario(ts[1], cfg, 2.0)], 500_000)
    assert cb.device_set is ts and cb.arrival is None
    assert list(cb.scenarios["trace_offset"]) == [ts.offsets[1], ts.offsets[0], ts.offsets[1]]
    assert list(cb.scenarios["n_requests"]) == [len(got[1][0]), len(got[0][0]), len(got[1][0])]
    host = compile_batch([Scenario(ts[1].to_host(), cfg, 0.5), Scenario(ts[0].to_host(), cfg, 1.0),
                          Scenario(ts[1].to_host(), cfg, 2.0)], 500_000)
    assert list(dispatch_order(cb)) == list(dispatch_order(host))
    assert arrow.native_rate(ts[0]) == arrow.native_rate(ts[0].to_host())
    # the KV bound is the one validation a generated trace can fail: same message as the host path
    tight = arrow.config_from_values(S.cfg(instances=4, kv_capacity_tokens=300, chunk_budget=128))
    with pytest.raises(ValueError) as dev:
        compile_batch([Scenario(ts[0], tight, 1.0)], 500_000)
    with pytest.raises(ValueError) as hst:
        compile_batch([Scenario(ts[0].to_host(), tight, 1.0)], 500_000)
    assert str(dev.value) == str(hst.value) and "KV tokens" in str(dev.value)
    with pytest.raises(ValueError, match="not a mix"):
        compile_batch([Scenario(ts[0], cfg, 1.0), Scenario(ts[0].to_host(), cfg, 1.0)], 500_000)
