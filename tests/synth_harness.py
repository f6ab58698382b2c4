"""Plumbing for the workload-generator parity tests (CPU and GPU).

Golden traces come from the real reference (oracle/gen_golden_traces.py ->
tests/golden/synth_traces.npz); random cases are checked against this
repo's numpy host generator (traces.gen_synthetic, itself pinned to the
golden vectors).  build/libnpgen_host.so is the device generator source
compiled for the host (test infrastructure only).
"""

from __future__ import annotations

import ctypes
import json
import math
import sys

import numpy as np

import harness as H
from paper_2505_11916_b200 import _abi
from paper_2505_11916_b200.traces import BurstEpisode, SyntheticParams

sys.path.insert(0, str(H.ROOT / "oracle"))
from synth_catalogue import catalogue  # noqa: E402

GOLDEN = H.GOLDEN / "synth_traces.npz"


def params_of(kw: dict) -> SyntheticParams:
    kw = dict(kw)
    kw["bursts"] = tuple(BurstEpisode(*b) for b in kw.get("bursts", ()))
    return SyntheticParams(**kw)


def golden_entries() -> list[tuple[str, SyntheticParams, tuple[np.ndarray, np.ndarray, np.ndarray]]]:
    z = np.load(GOLDEN)
    meta = json.loads(str(z["meta"]))
    errs = {e["name"]: e["error"] for e in meta["entries"]}
    out = []
    for name, kw in catalogue():
        assert errs[name] is None, (name, errs[name])
        out.append((name, params_of(kw), (z[f"{name}__arrival"], z[f"{name}__input"], z[f"{name}__output"])))
    return out


def random_params(rng: np.random.Generator) -> SyntheticParams:
    nb = int(rng.integers(0, 6))
    dur = float(rng.uniform(5.0, 120.0))
    bursts = tuple(
        BurstEpisode(float(rng.uniform(-10, dur)), float(rng.uniform(0.5, 40.0)), float(rng.choice([0.5, 1.5, 2.0, 4.0, 7.0])))
        for _ in range(nb)
    )
    return SyntheticParams(
        duration_s=dur,
        base_rate=float(rng.uniform(0.5, 20.0)),
        input_log_mean=float(rng.uniform(0.0, 8.0)),
        input_log_sigma=float(rng.uniform(0.0, 2.0)),
        output_log_mean=float(rng.uniform(0.0, 6.0)),
        output_log_sigma=float(rng.uniform(0.0, 2.0)),
        bursts=bursts,
        max_input=int(rng.integers(1, 20000)),
        max_output=int(rng.integers(1, 5000)),
        seed=int(rng.integers(0, 2**63)) >> int(rng.integers(0, 63)),
    )


def host_trace_arrays(params: SyntheticParams):
    from paper_2505_11916_b200.traces import gen_synthetic

    t = gen_synthetic(params)
    return (
        np.array([r.arrival for r in t], dtype=np.float64),
        np.array([r.input_len for r in t], dtype=np.int64),
        np.array([r.output_len for r in t], dtype=np.int64),
    )


def assert_trace_equal(name, got, exp) -> None:
    ga, gi, go = got
    ea, ei, eo = exp
    assert len(ga) == len(ea), f"{name}: {len(ga)} requests, reference {len(ea)}"
    if len(ea):
        bad = np.nonzero(np.asarray(ga, np.float64).view(np.uint64) != np.asarray(ea, np.float64).view(np.uint64))[0]
        assert bad.size == 0, f"{name}: arrival {bad[0]} differs: {ga[bad[0]]!r} vs {ea[bad[0]]!r}"
        assert np.array_equal(np.asarray(gi, np.int64), ei), f"{name}: input lengths differ"
        assert np.array_equal(np.asarray(go, np.int64), eo), f"{name}: output lengths differ"


def npgen_lib() -> ctypes.CDLL:
    if "npgen" not in H._libs:
        H._build("emu")
        lib = ctypes.CDLL(str(H.ROOT / "build" / "libnpgen_host.so"))
        lib.npgen_log1p.argtypes = [ctypes.c_double]
        lib.npgen_log1p.restype = ctypes.c_double
        lib.npgen_exp.argtypes = [ctypes.c_double]
        lib.npgen_exp.restype = ctypes.c_double
        lib.npgen_seed_state.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        lib.npgen_draw.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p]
        lib.npgen_check_libm.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_double)]
        lib.npgen_check_libm.restype = ctypes.c_int64
        lib.npgen_synth_run.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p]
        lib.npgen_synth_run.restype = ctypes.c_int
        H._libs["npgen"] = lib
    return H._libs["npgen"]


def host_emulated_batch(params_list):
    """The device generator source run on the host: list of (arrival, in, out)."""
    from paper_2505_11916_b200.device_traces import _capacity, synth_record

    lib = npgen_lib()
    specs = np.zeros(len(params_list), dtype=_abi.SYNTH_DTYPE)
    total = 0
    for i, p in enumerate(params_list):
        c = _capacity(p)
        specs[i] = synth_record(p, total, c)
        total += c
    arr = np.zeros(max(total, 1), dtype=np.float64)
    inp = np.zeros(max(total, 1), dtype=np.int32)
    outp = np.zeros(max(total, 1), dtype=np.int32)
    res = np.zeros(len(params_list), dtype=_abi.SYNTH_RESULT_DTYPE)
    lib.npgen_synth_run(specs.ctypes.data, len(params_list), arr.ctypes.data, inp.ctypes.data, outp.ctypes.data,
                        res.ctypes.data)
    out = []
    for i in range(len(params_list)):
        assert res["status"][i] == _abi.SYNTH_OK, (i, res[i])
        o, n = int(specs["out_offset"][i]), int(res["count"][i])
        out.append((arr[o : o + n], inp[o : o + n].astype(np.int64), outp[o : o + n].astype(np.int64)))
    return out, res


def seed_state_words(seed: int) -> list[int]:
    st = np.random.PCG64(seed).state["state"]
    m = (1 << 64) - 1
    return [st["state"] >> 64, st["state"] & m, st["inc"] >> 64, st["inc"] & m]


def isclose_bits(a: float, b: float) -> bool:
    return (math.isnan(a) and math.isnan(b)) or np.float64(a).tobytes() == np.float64(b).tobytes()
