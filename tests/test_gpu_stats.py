"""trace_stats on the B200.

Every golden case of the real reference: bucket totals, counts, duration,
rate, coefficients of variation and percentiles bit for bit; the Pearson r
within 1e-12 relative (numpy reaches it through BLAS, see stats.py).  Plus
seeded random traces against the CPU restatement, device-generated traces
read in place, and a 4 M-request trace through the radix-select path.
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np
import pytest

import synth_harness as SH
from test_stats_host import assert_stats_equal, golden_cases

import stats_oracle as SO  # noqa: E402  (oracle/ on sys.path via synth_harness)

pytestmark = pytest.mark.gpu


def _as_dict(s) -> dict:
    return dict(
        num_requests=s.num_requests, duration_s=s.duration_s, mean_rate=s.mean_rate,
        buckets=[[b.index, b.requests, b.input_tokens, b.output_tokens] for b in s.buckets],
        input_bucket_cv=s.input_bucket_cv, output_bucket_cv=s.output_bucket_cv, io_correlation=s.io_correlation,
        input_percentiles=s.input_percentiles, output_percentiles=s.output_percentiles,
    )


def _trace(a, i, o):
    from paper_2505_11916_b200 import TraceRequest

    return [TraceRequest(k, float(a[k]), int(i[k]), int(o[k])) for k in range(len(a))]


def test_golden_cases():
    import paper_2505_11916_b200 as arrow

    for c, (a, i, o) in golden_cases():
        s = arrow.trace_stats(_trace(a, i, o), bucket_s=c["bucket_s"])
        assert_stats_equal(_as_dict(s), c, c["name"], corr_rtol=1e-12)
        assert np.copysign(1.0, s.duration_s) == c["duration_sign"], c["name"]


def test_random_traces_vs_oracle():
    import paper_2505_11916_b200 as arrow

    rng = np.random.default_rng(202)
    for trial in range(30):
        n = int(rng.integers(1, 20000))
        a = np.sort(rng.uniform(0, float(rng.uniform(1, 5000)), n))
        if trial % 5 == 0:
            a = rng.permutation(a)
        hi = [50, 3000, 16384, 17000, 300000][trial % 5]
        i = rng.integers(1, hi + 1, n)
        o = rng.integers(1, max(2, hi // 3), n)
        b = float(rng.choice([0.05, 1.0, 7.5, 60.0, 1e4]))
        exp = SO.trace_stats_arrays(a, i, o, b)
        exp = dict(exp, input_percentiles={str(k): v for k, v in exp["input_percentiles"].items()},
                   output_percentiles={str(k): v for k, v in exp["output_percentiles"].items()})
        got = _as_dict(arrow.trace_stats(_trace(a, i, o), bucket_s=b))
        assert_stats_equal(got, exp, f"random[{trial}]", corr_rtol=1e-12)


def test_device_traces_in_place():
    import paper_2505_11916_b200 as arrow

    base = SH.params_of(dict(SH.catalogue())["bursty"])
    ts = arrow.gen_synthetic_batch([replace(base, seed=s) for s in (3, 4, 5)])
    for dt in ts:
        host = dt.to_host()
        for b in (1.0, 60.0):
            assert arrow.trace_stats(dt, bucket_s=b) == arrow.trace_stats(host, bucket_s=b)


def test_large_trace_radix_path():
    """4 M requests with lengths beyond the exact bins (two-level radix select)."""
    import paper_2505_11916_b200 as arrow
    from paper_2505_11916_b200 import stats as ST

    rng = np.random.default_rng(5)
    n = 4_000_000
    a = np.cumsum(rng.exponential(0.01, n))
    i = rng.integers(1, 1_000_000, n).astype(np.int32)
    o = rng.integers(1, 20_000, n).astype(np.int32)
    s = arrow.trace_stats(_trace(a[:10], i[:10], o[:10]), 1.0)  # warm
    # call through the device path on arrays (avoid 4 M Python objects): build a DeviceTrace-like view
    import torch

    from paper_2505_11916_b200.device_traces import DeviceTraceSet

    res = np.zeros(1, dtype=__import__("paper_2505_11916_b200")._abi.SYNTH_RESULT_DTYPE)
    res["count"], res["first_arrival"], res["last_arrival"] = n, a.min(), a.max()
    dev = torch.device("cuda")
    ts = DeviceTraceSet([None], torch.from_numpy(a).to(dev), torch.from_numpy(i).to(dev), torch.from_numpy(o).to(dev),
                        np.zeros(1, np.int64), res, dev)
    s = arrow.trace_stats(ts[0], bucket_s=60.0)
    assert s.num_requests == n
    for p in (50, 90, 99):
        assert s.input_percentiles[p] == int(np.percentile(i.astype(float), p))
        assert s.output_percentiles[p] == int(np.percentile(o.astype(float), p))
    lo = int(a.min() // 60.0)
    idx = (a // 60.0).astype(np.int64) - lo
    assert [b.requests for b in s.buckets] == np.bincount(idx, minlength=len(s.buckets)).tolist()
    assert [b.input_tokens for b in s.buckets] == np.bincount(idx, weights=i, minlength=len(s.buckets)).astype(
        np.int64).tolist()
    assert abs(s.io_correlation - float(np.corrcoef(i.astype(float), o.astype(float))[0, 1])) < 1e-12
    assert ST.HIST_BINS == 16384


def test_wrong_window_hint_is_rescanned():
    """The scan trusts the host's window (first/last arrival) to track min /
    max only in the edge buckets; a wrong window must be detected and
    rescanned to the exact answer."""
    import torch

    import paper_2505_11916_b200 as arrow
    from paper_2505_11916_b200 import stats as ST

    c, (a, i, o) = next((c, arrs) for c, arrs in golden_cases() if c["name"] == "bursty_7p5")
    trace = _trace(a, i, o)
    b = c["bucket_s"]
    dev = torch.device("cuda")
    stream = torch.cuda.current_stream(dev)
    lib = ST._lib()
    for lo_shift, hi_shift in ((2, 0), (0, -3), (-1, 2), (5, -5)):
        d = ST._Device(trace, dev)
        lo = int(d.first_hint // b) + lo_shift
        hi = int(d.last_hint // b) + hi_shift
        res = ST._run_scan(lib, torch, d, b, lo, hi - lo + 1, dev, stream)
        got = ST._finish(lib, torch, d, res, b, dev, stream)
        assert_stats_equal(_as_dict(got), c, f"window shifted {lo_shift},{hi_shift}", corr_rtol=1e-12)
    assert arrow.trace_stats(trace, b) == got
