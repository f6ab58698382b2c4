"""Trace statistics on the GPU: ``trace_stats``.

Drop-in for ``pdsim.traces.trace_stats`` (traces.py:202-250).  The
per-request scan (16 B per request: bucket totals, length histograms,
integer moments, first/last arrival) is one pass of the sm_100a kernel in
csrc/stats.cu; the host turns its O(buckets + 16 K) outputs into the
reference's ``TraceStats`` with the reference's own formulas:

* buckets: exact integer totals; ``int(arrival // bucket_s)`` is CPython's
  float floor division, reproduced on the device;
* ``input_bucket_cv`` / ``output_bucket_cv``: numpy ``std / mean`` over the
  (exact) bucket totals, as the reference computes them -> bit-identical;
* ``input_percentiles`` / ``output_percentiles``: np.percentile's linear
  interpolation between exact order statistics (device histograms, plus a
  two-level device radix select for lengths above 16 384) -> bit-identical;
* ``io_correlation``: the Pearson r from exact 128-bit integer moments,
  correctly rounded up to the final division / square root.  numpy gets it
  through BLAS (``np.corrcoef``), whose summation order is not specified,
  so this field agrees to ~1e-15 relative, not bit for bit.

There is no CPU fallback: without a GPU or the built library this raises.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from .core import TraceRequest

HIST_BINS = 16384
MAX_BUCKETS = 1 << 28

PARTIAL_DTYPE = np.dtype(
    [
        ("min_arrival", np.float64),
        ("max_arrival", np.float64),
        ("count", np.int64),
        ("sum_x", np.int64),
        ("sum_y", np.int64),
        ("sxx_lo", np.uint64),
        ("sxx_hi", np.uint64),
        ("syy_lo", np.uint64),
        ("syy_hi", np.uint64),
        ("sxy_lo", np.uint64),
        ("sxy_hi", np.uint64),
        ("out_of_window", np.int64),
    ],
    align=True,
)


class StatsArgs(ctypes.Structure):
    """arrow_stats_args_t (include/arrow_traces.h)."""

    _fields_ = [
        ("arrival", ctypes.c_void_p),
        ("input_len", ctypes.c_void_p),
        ("output_len", ctypes.c_void_p),
        ("n", ctypes.c_int64),
        ("bucket_s", ctypes.c_double),
        ("bucket_lo", ctypes.c_int64),
        ("n_buckets", ctypes.c_int64),
        ("bucket_requests", ctypes.c_void_p),
        ("bucket_input", ctypes.c_void_p),
        ("bucket_output", ctypes.c_void_p),
        ("hist_x", ctypes.c_void_p),
        ("hist_y", ctypes.c_void_p),
        ("partials", ctypes.c_void_p),
        ("n_partials", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


@dataclass(frozen=True)
class BucketStats:
    index: int
    requests: int
    input_tokens: int
    output_tokens: int


@dataclass(frozen=True)
class TraceStats:
    num_requests: int
    duration_s: float
    mean_rate: float
    buckets: tuple[BucketStats, ...]
    input_bucket_cv: float
    output_bucket_cv: float
    io_correlation: float
    input_percentiles: dict[int, int] = field(default_factory=dict)
    output_percentiles: dict[int, int] = field(default_factory=dict)


_ready = False


def _lib():
    global _ready
    from ._backend import load_library

    lib = load_library()
    if not _ready:
        lib.arrow_stats_grid.argtypes = [ctypes.c_int64, ctypes.POINTER(ctypes.c_int32)]
        lib.arrow_stats_grid.restype = ctypes.c_int
        lib.arrow_stats_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        lib.arrow_stats_run.restype = ctypes.c_int
        lib.arrow_stats_hist.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        lib.arrow_stats_hist.restype = ctypes.c_int
        _ready = True
    return lib


def percentile_from_order(n: int, order_stat, p: int) -> int:
    """``int(np.percentile(values, p))`` (method "linear") from the order
    statistics of ``values`` (``order_stat(k)`` = k-th smallest, 0-based):
    numpy's virtual index, clipping and _lerp, in float64."""
    q = np.true_divide(p, 100)
    virtual = (n - 1) * q
    if virtual >= n - 1:
        prev_i, next_i, prev_f = n - 1, n - 1, np.intp(-1)
    elif virtual < 0:
        prev_i, next_i, prev_f = 0, 0, np.intp(0)
    else:
        prev_i = int(np.floor(virtual))
        next_i = prev_i + 1
        prev_f = np.intp(prev_i)
    gamma = np.float64(virtual - prev_f)
    a = np.float64(order_stat(prev_i))
    b = np.float64(order_stat(next_i))
    diff = b - a
    lerp = a + diff * gamma
    if gamma >= 0.5:
        lerp = b - diff * (1 - gamma)
    return int(lerp)


def _cv(values: list[int]) -> float:
    """traces.py:231-234, verbatim numpy."""
    arr = np.array(values, dtype=float)
    mean = arr.mean()
    return float(arr.std() / mean) if mean > 0 else 0.0


def _u128(lo, hi) -> int:
    return int(lo) | (int(hi) << 64)


def _floordiv_index(x: float, b: float) -> int:
    return int(x // b)


class _Device:
    """Device views of one trace's SoA arrays (uploaded or generated)."""

    def __init__(self, trace, device):
        import torch

        from .device_traces import DeviceTrace

        self.torch = torch
        self.h2d = 0
        if isinstance(trace, DeviceTrace):
            s = slice(trace.offset, trace.offset + trace.n)
            self.arrival = trace.set.arrival[s]
            self.input_len = trace.set.input_len[s]
            self.output_len = trace.set.output_len[s]
            self.n = trace.n
            self.first_hint, self.last_hint = trace.first_arrival, trace.last_arrival
        else:
            from .traces import trace_arrays

            a, i, o = trace_arrays(trace)
            self.n = len(a)
            self.first_hint, self.last_hint = float(a.min()), float(a.max())
            pa = torch.from_numpy(a).pin_memory()
            pi = torch.from_numpy(i).pin_memory()
            po = torch.from_numpy(o).pin_memory()
            self.arrival = pa.to(device, non_blocking=True)
            self.input_len = pi.to(device, non_blocking=True)
            self.output_len = po.to(device, non_blocking=True)
            self.h2d = a.nbytes + i.nbytes + o.nbytes


def _order_stats(lib, torch, values_dev, hist: np.ndarray, over: int, n: int, ranks, device, stream):
    """k-th smallest lengths for every k in ranks: exact bins 1..16384, then a
    two-level device radix select over the values above (up to 2^31 - 1)."""
    cum = np.cumsum(hist.astype(np.int64))
    in_bins = int(cum[-1])
    assert in_bins + over == n
    out = {}
    need_high = []
    for k in ranks:
        if k < in_bins:
            out[k] = int(np.searchsorted(cum, k, side="right")) + 1
        else:
            need_high.append(k)
    if not need_high:
        return out
    lo, hi = HIST_BINS + 1, 1 << 31
    shift = max(0, (hi - lo - 1).bit_length() - 20)
    nb = ((hi - lo - 1) >> shift) + 1
    bins = torch.empty(nb, dtype=torch.int32, device=device)
    rc = lib.arrow_stats_hist(values_dev.data_ptr(), n, lo, hi, shift, bins.data_ptr(), nb,
                              ctypes.c_void_p(stream.cuda_stream))
    if rc:
        raise RuntimeError(f"arrow_stats_hist failed: cuda error {rc}")
    c1 = np.cumsum(bins.cpu().numpy().view(np.uint32).astype(np.int64))
    for k in need_high:
        r = k - in_bins
        j = int(np.searchsorted(c1, r, side="right"))
        before = int(c1[j - 1]) if j else 0
        if shift == 0:
            out[k] = lo + j
            continue
        blo = lo + (j << shift)
        bhi = min(blo + (1 << shift), hi)
        fine = torch.empty(bhi - blo, dtype=torch.int32, device=device)
        rc = lib.arrow_stats_hist(values_dev.data_ptr(), n, blo, bhi, 0, fine.data_ptr(), bhi - blo,
                                  ctypes.c_void_p(stream.cuda_stream))
        if rc:
            raise RuntimeError(f"arrow_stats_hist failed: cuda error {rc}")
        c2 = np.cumsum(fine.cpu().numpy().view(np.uint32).astype(np.int64))
        out[k] = blo + int(np.searchsorted(c2, r - before, side="right"))
    return out


def trace_stats(trace, bucket_s: float = 60.0, device=None, stream=None) -> TraceStats:
    """Per-bucket arrival totals plus dispersion / correlation / percentile
    numbers of a trace (traces.py:202-250).  ``trace`` is a list of
    TraceRequest or a device_traces.DeviceTrace (read in place)."""
    import torch

    from ._backend import EvaluatorUnavailable

    if isinstance(trace, list) and not trace or (not isinstance(trace, list) and len(trace) == 0):
        raise ValueError("empty trace")
    if bucket_s <= 0:
        raise ValueError("bucket_s must be positive")
    if not torch.cuda.is_available():
        raise EvaluatorUnavailable("no CUDA device: trace_stats runs only on the GPU (no CPU fallback)")
    lib = _lib()
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    stream = stream if stream is not None else torch.cuda.current_stream(device)
    with torch.cuda.device(device):
        d = _Device(trace, device)
        lo = _floordiv_index(d.first_hint, bucket_s)
        hi = _floordiv_index(d.last_hint, bucket_s)
        nb = hi - lo + 1
        if nb > MAX_BUCKETS or abs(lo) >= 2**53:
            raise ValueError(f"{nb} buckets of {bucket_s} s exceed the device limit of {MAX_BUCKETS}")
        res = _run_scan(lib, torch, d, bucket_s, lo, nb, device, stream)
        return _finish(lib, torch, d, res, bucket_s, device, stream)


def _run_scan(lib, torch, d, bucket_s, lo, nb, device, stream):
    grid = ctypes.c_int32(0)
    lib.arrow_stats_grid(d.n, ctypes.byref(grid))
    g = grid.value
    bk = torch.empty((3, max(nb, 1)), dtype=torch.int64, device=device)
    hist = torch.empty((2, HIST_BINS), dtype=torch.int32, device=device)
    parts = torch.empty(g * PARTIAL_DTYPE.itemsize, dtype=torch.uint8, device=device)
    a = StatsArgs(
        d.arrival.data_ptr(), d.input_len.data_ptr(), d.output_len.data_ptr(), d.n, float(bucket_s), lo, nb,
        bk[0].data_ptr(), bk[1].data_ptr(), bk[2].data_ptr(), hist[0].data_ptr(), hist[1].data_ptr(),
        parts.data_ptr(), g, 0,
    )
    rc = lib.arrow_stats_run(ctypes.addressof(a), ctypes.c_void_p(stream.cuda_stream))
    if rc:
        raise RuntimeError(f"arrow_stats_run failed: cuda error {rc}")
    p = np.frombuffer(parts.cpu().numpy().tobytes(), dtype=PARTIAL_DTYPE)
    return dict(lo=lo, nb=nb, buckets=bk.cpu().numpy(), hist=hist.cpu().numpy().view(np.uint32), partials=p)


def _merge(p: np.ndarray) -> dict:
    """Fold the per-block partials.  first/last: min/max arrival (Python's
    min/max would return the first of equal values, which can differ only in
    the sign of a zero -- unobservable in TraceStats, see csrc/stats.cu)."""
    live = p[~np.isnan(p["min_arrival"])]
    return dict(
        n=int(live["count"].sum()),
        first=float(live["min_arrival"].min()),
        last=float(live["max_arrival"].max()),
        sx=int(live["sum_x"].astype(object).sum()),
        sy=int(live["sum_y"].astype(object).sum()),
        sxx=sum(_u128(r["sxx_lo"], r["sxx_hi"]) for r in live),
        syy=sum(_u128(r["syy_lo"], r["syy_hi"]) for r in live),
        sxy=sum(_u128(r["sxy_lo"], r["sxy_hi"]) for r in live),
        oow=int(live["out_of_window"].sum()),
    )


def pearson_from_moments(n: int, sx: int, sy: int, sxx: int, syy: int, sxy: int) -> float:
    """Pearson r of exact integer moments, clipped like np.corrcoef."""
    num = n * sxy - sx * sy
    dx = n * sxx - sx * sx
    dy = n * syy - sy * sy
    if dx <= 0 or dy <= 0:
        return 0.0
    # num / sqrt(dx * dy) evaluated with a 128-bit-scaled integer square
    # root, then rounded once to float
    k = 128
    r = float(Fraction(num << k, math.isqrt((dx * dy) << (2 * k))))
    return float(min(1.0, max(-1.0, r)))


def _finish(lib, torch, d, res, bucket_s, device, stream) -> TraceStats:
    m = _merge(res["partials"])
    lo = _floordiv_index(m["first"], bucket_s)
    hi = _floordiv_index(m["last"], bucket_s)
    for _ in range(3):
        if not m["oow"] and lo == res["lo"] and hi - lo + 1 == res["nb"]:
            break
        # the window hint disagreed with the data (cannot happen for exact
        # hints): rescan with the window of the scanned first / last arrival
        res = _run_scan(lib, torch, d, bucket_s, lo, hi - lo + 1, device, stream)
        m = _merge(res["partials"])
        lo = _floordiv_index(m["first"], bucket_s)
        hi = _floordiv_index(m["last"], bucket_s)
    assert m["n"] == d.n and not m["oow"], (m["n"], d.n, m["oow"])
    bk = res["buckets"]
    buckets = tuple(
        BucketStats(lo + j, int(bk[0, j]), int(bk[1, j]), int(bk[2, j])) for j in range(hi - lo + 1)
    )
    n = m["n"]
    duration = m["last"] - m["first"]
    ranks = {0, n - 1}  # min / max: the std > 0 tests of traces.py:238
    for p in (50, 90, 99):
        v = (n - 1) * np.true_divide(p, 100)
        f = int(np.floor(v))
        ranks.update(k for k in (f, f + 1) if 0 <= k < n)
    # lengths outside the exact bins: n - sum(bins)
    over_x = n - int(res["hist"][0].astype(np.int64).sum())
    over_y = n - int(res["hist"][1].astype(np.int64).sum())
    osx = _order_stats(lib, torch, d.input_len, res["hist"][0], over_x, n, sorted(ranks), device, stream)
    osy = _order_stats(lib, torch, d.output_len, res["hist"][1], over_y, n, sorted(ranks), device, stream)
    # inputs.std() > 0 and outputs.std() > 0 <=> neither array is constant
    if n >= 2 and osx[0] != osx[n - 1] and osy[0] != osy[n - 1]:
        corr = pearson_from_moments(n, m["sx"], m["sy"], m["sxx"], m["syy"], m["sxy"])
    else:
        corr = 0.0
    return TraceStats(
        num_requests=n,
        duration_s=duration,
        mean_rate=(n - 1) / duration if duration > 0 else math.inf,
        buckets=buckets,
        input_bucket_cv=_cv([b.input_tokens for b in buckets]),
        output_bucket_cv=_cv([b.output_tokens for b in buckets]),
        io_correlation=corr,
        input_percentiles={p: percentile_from_order(n, osx.__getitem__, p) for p in (50, 90, 99)},
        output_percentiles={p: percentile_from_order(n, osy.__getitem__, p) for p in (50, 90, 99)},
    )
