"""Workload generation feeding the evaluator (mirrors pdsim.traces).

The generator consumes numpy's PCG64 stream in exactly the reference's call
order (traces.py:159-175: exponential gap, thinning uniform, two normals per
accepted arrival), so a seed yields the same trace bit for bit.  Traces are
shipped to the GPU as struct-of-arrays (arrival f64, input i32, output i32)
by :func:`trace_arrays`.
"""

from __future__ import annotations

import csv
import json
import math
from dataclasses import dataclass
from operator import attrgetter
from pathlib import Path

import numpy as np

from .core import TraceRequest

_FIELDS = ("arrival_s", "input_tokens", "output_tokens")


class TraceFormatError(ValueError):
    pass


@dataclass(frozen=True)
class BurstEpisode:
    """Rate multiplier on [start, start + duration)."""

    start: float
    duration: float
    multiplier: float

    def __post_init__(self) -> None:
        if self.duration <= 0 or self.multiplier <= 0:
            raise ValueError("burst duration and multiplier must be positive")


@dataclass(frozen=True)
class SyntheticParams:
    """Thinned Poisson arrivals with bursts, log-normal lengths."""

    duration_s: float
    base_rate: float
    input_log_mean: float
    input_log_sigma: float
    output_log_mean: float
    output_log_sigma: float
    bursts: tuple[BurstEpisode, ...] = ()
    max_input: int = 16384
    max_output: int = 4096
    seed: int = 0

    def __post_init__(self) -> None:
        if self.duration_s < 0:
            raise ValueError("duration_s must be >= 0")
        if self.base_rate <= 0:
            raise ValueError("base_rate must be positive")
        if min(self.input_log_sigma, self.output_log_sigma) < 0:
            raise ValueError("log sigmas must be >= 0")


def _intensity(params: SyntheticParams, t: float) -> float:
    rate = params.base_rate
    for ep in params.bursts:
        if ep.start <= t < ep.start + ep.duration:
            rate *= ep.multiplier
    return rate


def _lognormal_len(rng: np.random.Generator, mu: float, sigma: float, cap: int) -> int:
    value = round(math.exp(rng.normal(mu, sigma)))
    return int(min(max(value, 1), cap))


def gen_synthetic(params: SyntheticParams) -> list[TraceRequest]:
    rng = np.random.default_rng(params.seed)
    peak = params.base_rate * max((ep.multiplier for ep in params.bursts), default=1.0)
    out: list[TraceRequest] = []
    t = 0.0
    while True:
        t += rng.exponential(1.0 / peak)
        if t >= params.duration_s:
            return out
        if rng.random() * peak > _intensity(params, t):
            continue
        n_in = _lognormal_len(rng, params.input_log_mean, params.input_log_sigma, params.max_input)
        n_out = _lognormal_len(rng, params.output_log_mean, params.output_log_sigma, params.max_output)
        out.append(TraceRequest(len(out), float(t), n_in, n_out))


def native_rate(trace: list[TraceRequest]) -> float:
    """(n - 1) / span, the reference rate for rescaling (traces.py:253-261)."""
    if hasattr(trace, "native_rate"):  # device_traces.DeviceTrace: from its device-side summary
        return trace.native_rate()
    if len(trace) < 2:
        raise ValueError("need at least 2 requests to define a rate")
    span = trace[-1].arrival - trace[0].arrival
    if span <= 0:
        raise ValueError("trace span must be positive to define a rate")
    return (len(trace) - 1) / span


def bundled_bursty_trace() -> list[TraceRequest]:
    """2 606-request bursty workload (traces.py:267-286)."""
    return gen_synthetic(
        SyntheticParams(
            duration_s=360.0,
            base_rate=4.0,
            input_log_mean=math.log(420.0),
            input_log_sigma=0.55,
            output_log_mean=math.log(130.0),
            output_log_sigma=0.5,
            bursts=(BurstEpisode(50.0, 25.0, 5.0), BurstEpisode(150.0, 30.0, 4.0), BurstEpisode(260.0, 25.0, 5.0)),
            max_input=3500,
            max_output=900,
            seed=20240817,
        )
    )


def bundled_ramp_trace() -> list[TraceRequest]:
    """686-request ramp workload (traces.py:289-309)."""
    return gen_synthetic(
        SyntheticParams(
            duration_s=300.0,
            base_rate=1.0,
            input_log_mean=math.log(500.0),
            input_log_sigma=0.4,
            output_log_mean=math.log(350.0),
            output_log_sigma=0.35,
            bursts=(
                BurstEpisode(60.0, 40.0, 2.0),
                BurstEpisode(100.0, 40.0, 4.0),
                BurstEpisode(140.0, 40.0, 6.0),
                BurstEpisode(180.0, 30.0, 3.0),
            ),
            max_input=3000,
            max_output=1200,
            seed=7,
        )
    )


def trace_arrays(trace: list[TraceRequest]) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Struct-of-arrays view of a trace: (arrival f64, input i32, output i32)."""
    n = len(trace)
    arrival = np.fromiter(map(_ARRIVAL, trace), dtype=np.float64, count=n)
    inp = np.fromiter(map(_INPUT, trace), dtype=np.int32, count=n)
    outp = np.fromiter(map(_OUTPUT, trace), dtype=np.int32, count=n)
    return arrival, inp, outp


_ARRIVAL, _INPUT, _OUTPUT = attrgetter("arrival"), attrgetter("input_len"), attrgetter("output_len")


# -- canonical file formats (traces.py:23-102) -----------------------------


def _from_rows(rows: list[tuple[float, int, int]], source: str) -> list[TraceRequest]:
    order = sorted(range(len(rows)), key=lambda i: (rows[i][0], i))
    trace = []
    for new_id, i in enumerate(order):
        try:
            trace.append(TraceRequest(new_id, *rows[i]))
        except ValueError as exc:
            raise TraceFormatError(f"{source}: record {i + 1}: {exc}") from exc
    return trace


def load_trace(path: str | Path, fmt: str | None = None) -> list[TraceRequest]:
    path = Path(path)
    fmt = fmt or ("csv" if path.suffix.lower() == ".csv" else "jsonl")
    if fmt not in ("jsonl", "csv"):
        raise TraceFormatError(f"unsupported trace format {fmt!r}")
    rows: list[tuple[float, int, int]] = []
    with open(path, newline="") as f:
        if fmt == "jsonl":
            for lineno, line in enumerate(f, start=1):
                if not line.strip():
                    continue
                try:
                    obj = json.loads(line)
                    rows.append((float(obj[_FIELDS[0]]), int(obj[_FIELDS[1]]), int(obj[_FIELDS[2]])))
                except (json.JSONDecodeError, KeyError, TypeError, ValueError) as exc:
                    raise TraceFormatError(f"{path}:{lineno}: {exc}") from exc
        else:
            reader = csv.DictReader(f)
            if reader.fieldnames is None or [c.strip() for c in reader.fieldnames] != list(_FIELDS):
                raise TraceFormatError(f"{path}: expected header {','.join(_FIELDS)}, got {reader.fieldnames}")
            for lineno, row in enumerate(reader, start=2):
                try:
                    rows.append((float(row[_FIELDS[0]]), int(row[_FIELDS[1]]), int(row[_FIELDS[2]])))
                except (TypeError, ValueError) as exc:
                    raise TraceFormatError(f"{path}:{lineno}: {exc}") from exc
    return _from_rows(rows, str(path))


def save_trace(trace: list[TraceRequest], path: str | Path, fmt: str | None = None) -> None:
    path = Path(path)
    fmt = fmt or ("csv" if path.suffix.lower() == ".csv" else "jsonl")
    ordered = sorted(trace, key=lambda r: (r.arrival, r.id))
    if fmt == "jsonl":
        with open(path, "w") as f:
            for r in ordered:
                f.write(json.dumps(dict(zip(_FIELDS, (r.arrival, r.input_len, r.output_len)))) + "\n")
    elif fmt == "csv":
        with open(path, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(_FIELDS)
            w.writerows([repr(float(r.arrival)), r.input_len, r.output_len] for r in ordered)
    else:
        raise TraceFormatError(f"unsupported trace format {fmt!r}")


# traces.trace_stats (traces.py:181-250) lives with its GPU scan in stats.py
from .stats import BucketStats, TraceStats, trace_stats  # noqa: E402,F401
