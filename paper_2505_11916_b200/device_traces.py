"""Device workload generator.

``gen_synthetic_batch(params)`` runs the reference's generator
(``pdsim.traces.gen_synthetic``, traces.py:159-175) for a whole list of
``SyntheticParams`` (typically one per seed) in one CUDA launch, bit for bit:
numpy's ``default_rng(seed)`` SeedSequence + PCG64 stream, its ziggurat
exponential / normal samplers, glibc's ``exp``/``log1p`` and CPython's
``round`` are restated in ``csrc/npgen.cuh``.  The traces stay in device
memory, laid out as the evaluator's struct-of-arrays trace table, so a
multi-seed sweep never ships traces over PCIe:

    traces = gen_synthetic_batch([replace(p, seed=s) for s in seeds])
    hb = evaluate_scenarios([Scenario(traces[i], cfg, scale) for ...])

``DeviceTrace.to_host()`` returns the reference's ``list[TraceRequest]``.
There is no CPU fallback: without a GPU or the built library this raises.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _abi
from .core import TraceRequest
from .traces import SyntheticParams


def seed_words(seed) -> list[int]:
    """SeedSequence entropy of ``default_rng(seed)`` for an int seed: its
    little-endian uint32 words (numpy's _int_to_uint32_array); ``None`` draws
    fresh OS entropy exactly as numpy does."""
    if seed is None:
        seed = np.random.SeedSequence().entropy
    if isinstance(seed, (bool, np.bool_)) or not isinstance(seed, (int, np.integer)):
        raise TypeError(f"the device generator takes integer seeds, got {type(seed).__name__}")
    seed = int(seed)
    if seed < 0:
        raise ValueError("expected non-negative integer")
    if seed == 0:
        return [0]
    words = []
    while seed:
        words.append(seed & 0xFFFFFFFF)
        seed >>= 32
    if len(words) > _abi.SYNTH_MAX_SEED_WORDS:
        raise ValueError(f"seeds above 2**{32 * _abi.SYNTH_MAX_SEED_WORDS} are not supported by the device generator")
    return words


def expected_requests(params: SyntheticParams) -> float:
    """Integral of the thinned intensity over [0, duration): the mean trace length."""
    d = float(params.duration_s)
    cuts = {0.0, d}
    for ep in params.bursts:
        for x in (ep.start, ep.start + ep.duration):
            if 0.0 < x < d:
                cuts.add(float(x))
    pts = sorted(cuts)
    total = 0.0
    for a, b in zip(pts, pts[1:]):
        mid = 0.5 * (a + b)
        rate = params.base_rate
        for ep in params.bursts:
            if ep.start <= mid < ep.start + ep.duration:
                rate *= ep.multiplier
        total += rate * (b - a)
    return total


def synth_record(params: SyntheticParams, out_offset: int, capacity: int) -> np.void:
    if not math.isfinite(params.duration_s):
        raise ValueError("the device generator needs a finite duration_s")
    if len(params.bursts) > _abi.SYNTH_MAX_BURSTS:
        raise ValueError(f"at most {_abi.SYNTH_MAX_BURSTS} burst episodes are supported by the device generator")
    for name in ("max_input", "max_output"):
        if getattr(params, name) > 2**31 - 1:
            raise ValueError(f"{name} above 2**31 - 1 is not supported by the device generator")
    words = seed_words(params.seed)
    rec = np.zeros((), dtype=_abi.SYNTH_DTYPE)
    # traces.py:162, 166 evaluated with Python floats
    rate_max = params.base_rate * max((ep.multiplier for ep in params.bursts), default=1.0)
    rec["duration_s"] = params.duration_s
    rec["base_rate"] = params.base_rate
    rec["rate_max"] = rate_max
    rec["gap_scale"] = 1.0 / rate_max
    rec["input_log_mean"], rec["input_log_sigma"] = params.input_log_mean, params.input_log_sigma
    rec["output_log_mean"], rec["output_log_sigma"] = params.output_log_mean, params.output_log_sigma
    rec["max_input"], rec["max_output"] = params.max_input, params.max_output
    rec["n_bursts"] = len(params.bursts)
    rec["n_seed_words"] = len(words)
    rec["seed_words"][: len(words)] = words
    for b, ep in enumerate(params.bursts):
        rec["burst_start"][b] = ep.start
        rec["burst_duration"][b] = ep.duration
        rec["burst_multiplier"][b] = ep.multiplier
    rec["out_offset"] = out_offset
    rec["capacity"] = capacity
    return rec


def _capacity(params: SyntheticParams) -> int:
    lam = expected_requests(params)
    return _round4(int(lam + 10.0 * math.sqrt(lam) + 32))


def _round4(c: int) -> int:
    """Slots per trace in multiples of 4 requests, so every trace's slice of
    the SoA arrays starts 16-byte aligned (TMA bulk copies in stats.cu)."""
    return (int(c) + 3) // 4 * 4


_lib_ready = False


def _load():
    global _lib_ready
    from ._backend import load_library

    lib = load_library()
    if not _lib_ready:
        lib.arrow_synth_run.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.arrow_synth_run.restype = ctypes.c_int
        _lib_ready = True
    return lib


class DeviceTrace:
    """One generated trace, resident on the device (a slice of its set)."""

    def __init__(self, tset: "DeviceTraceSet", index: int) -> None:
        self.set = tset
        self.index = index
        r = tset.results[index]
        self.offset = int(tset.offsets[index])
        self.n = int(r["count"])
        self.first_arrival = float(r["first_arrival"])
        self.last_arrival = float(r["last_arrival"])
        self.max_kv = int(r["max_kv"])
        self.sum_output = int(r["sum_output"])

    def __len__(self) -> int:
        return self.n

    def native_rate(self) -> float:
        """traces.py:253-261 from the device-side first/last arrival."""
        if self.n < 2:
            raise ValueError("need at least 2 requests to define a rate")
        span = self.last_arrival - self.first_arrival
        if span <= 0:
            raise ValueError("trace span must be positive to define a rate")
        return (self.n - 1) / span

    def arrays(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(arrival f64, input i32, output i32) copied to the host."""
        s = slice(self.offset, self.offset + self.n)
        return (
            self.set.arrival[s].cpu().numpy(),
            self.set.input_len[s].cpu().numpy(),
            self.set.output_len[s].cpu().numpy(),
        )

    def to_host(self) -> list[TraceRequest]:
        a, i, o = self.arrays()
        return [TraceRequest(k, float(a[k]), int(i[k]), int(o[k])) for k in range(self.n)]


class DeviceTraceSet:
    """Traces generated by one launch; trace i occupies
    [offsets[i], offsets[i] + counts[i]) of the SoA arrays."""

    def __init__(self, params, arrival, input_len, output_len, offsets, results, device) -> None:
        self.params = list(params)
        self.arrival = arrival
        self.input_len = input_len
        self.output_len = output_len
        self.offsets = offsets
        self.results = results
        self.device = device
        self.traces = [DeviceTrace(self, i) for i in range(len(self.params))]

    def __len__(self) -> int:
        return len(self.traces)

    def __getitem__(self, i: int) -> DeviceTrace:
        return self.traces[i]

    @property
    def counts(self) -> np.ndarray:
        return self.results["count"].astype(np.int64)

    def to_host(self) -> list[list[TraceRequest]]:
        return [t.to_host() for t in self.traces]


def _launch(lib, torch, specs: np.ndarray, total: int, device, stream):
    n = len(specs)
    arrival = torch.empty(max(total, 1), dtype=torch.float64, device=device)
    inp = torch.empty(max(total, 1), dtype=torch.int32, device=device)
    outp = torch.empty(max(total, 1), dtype=torch.int32, device=device)
    d_specs = torch.from_numpy(specs.view(np.uint8).reshape(-1).copy()).to(device)
    d_res = torch.empty(max(n, 1) * _abi.SYNTH_RESULT_DTYPE.itemsize, dtype=torch.uint8, device=device)
    s = stream if stream is not None else torch.cuda.current_stream(device)
    with torch.cuda.device(device):
        rc = lib.arrow_synth_run(d_specs.data_ptr(), n, arrival.data_ptr(), inp.data_ptr(), outp.data_ptr(),
                                 d_res.data_ptr(), ctypes.c_void_p(s.cuda_stream))
    if rc:
        raise RuntimeError(f"arrow_synth_run failed: cuda error {rc}")
    res = np.frombuffer(d_res[: n * _abi.SYNTH_RESULT_DTYPE.itemsize].cpu().numpy().tobytes(),
                        dtype=_abi.SYNTH_RESULT_DTYPE)
    return arrival, inp, outp, res


def gen_synthetic_batch(params_list, device=None, stream=None) -> DeviceTraceSet:
    """Generate every trace of ``params_list`` on the GPU (one thread per
    trace); equal, element for element, to ``[gen_synthetic(p) for p in
    params_list]`` of the reference."""
    import torch

    from ._backend import EvaluatorUnavailable

    if not torch.cuda.is_available():
        raise EvaluatorUnavailable("no CUDA device: the trace generator runs only on the GPU (no CPU fallback)")
    params_list = list(params_list)
    lib = _load()
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    caps = [_capacity(p) for p in params_list]
    for _attempt in range(2):
        offsets = np.zeros(len(params_list), dtype=np.int64)
        specs = np.zeros(len(params_list), dtype=_abi.SYNTH_DTYPE)
        total = 0
        for i, (p, c) in enumerate(zip(params_list, caps)):
            offsets[i] = total
            specs[i] = synth_record(p, total, c)
            total += c
        arrival, inp, outp, res = _launch(lib, torch, specs, total, device, stream)
        over = res["status"] == _abi.SYNTH_CAPACITY
        if not over.any():
            break
        caps = [_round4(max(c, n)) for c, n in zip(caps, res["count"])]
    for i, p in enumerate(params_list):
        r = res[i]
        if int(r["count"]) > 0:
            # TraceRequest.__post_init__ (core.py:46-52) on the first request
            if p.max_input < 1:
                raise ValueError(f"input_len must be >= 1, got {p.max_input}")
            if p.max_output < 1:
                raise ValueError(f"output_len must be >= 1, got {p.max_output}")
        if int(r["status"]) == _abi.SYNTH_OVERFLOW:
            raise OverflowError("math range error")  # math.exp, traces.py:155
    return DeviceTraceSet(params_list, arrival, inp, outp, offsets, res, device)
