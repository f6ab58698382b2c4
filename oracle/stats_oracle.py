"""CPU restatement of the reference's trace_stats (TEST INFRASTRUCTURE).

Follows /root/reference/pkg/src/pdsim/traces.py:202-250 line for line on
numpy arrays instead of TraceRequest objects, so the GPU tests can check
random traces on a box without the reference.  Pinned against the real
reference by tests/test_stats_host.py (golden file tests/golden/trace_stats.json
written by oracle/gen_golden_stats.py).  Only tests import this module.
"""

from __future__ import annotations

import math

import numpy as np


def trace_stats_arrays(arrival, input_len, output_len, bucket_s: float = 60.0) -> dict:
    n = len(arrival)
    if n == 0:
        raise ValueError("empty trace")                       # traces.py:211-212
    if bucket_s <= 0:
        raise ValueError("bucket_s must be positive")         # traces.py:213-214
    arr_list = [float(a) for a in arrival]
    first = min(arr_list)                                     # traces.py:215-216
    last = max(arr_list)
    lo = int(first // bucket_s)
    hi = int(last // bucket_s)
    totals = {i: [0, 0, 0] for i in range(lo, hi + 1)}       # traces.py:219-224
    for a, x, y in zip(arr_list, input_len, output_len):
        b = totals[int(a // bucket_s)]
        b[0] += 1
        b[1] += int(x)
        b[2] += int(y)
    buckets = [(i, *totals[i]) for i in range(lo, hi + 1)]

    def cv(values):                                           # traces.py:231-234
        arr = np.array(values, dtype=float)
        mean = arr.mean()
        return float(arr.std() / mean) if mean > 0 else 0.0

    inputs = np.array([int(v) for v in input_len], dtype=float)   # traces.py:236-241
    outputs = np.array([int(v) for v in output_len], dtype=float)
    if n >= 2 and inputs.std() > 0 and outputs.std() > 0:
        corr = float(np.corrcoef(inputs, outputs)[0, 1])
    else:
        corr = 0.0
    duration = last - first                                   # traces.py:242-250
    return dict(
        num_requests=n,
        duration_s=duration,
        mean_rate=(n - 1) / duration if duration > 0 else math.inf,
        buckets=buckets,
        input_bucket_cv=cv([b[2] for b in buckets]),
        output_bucket_cv=cv([b[3] for b in buckets]),
        io_correlation=corr,
        input_percentiles={p: int(np.percentile(inputs, p)) for p in (50, 90, 99)},
        output_percentiles={p: int(np.percentile(outputs, p)) for p in (50, 90, 99)},
    )
