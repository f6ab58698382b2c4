"""trace_stats host logic, checked WITHOUT a GPU.

* oracle/stats_oracle.py (the CPU restatement used by the GPU tests) equals
  the real reference on every golden case;
* the host finalisation the GPU path uses -- np.percentile from order
  statistics, the Pearson r from exact integer moments, the merge of
  per-block partials -- reproduces numpy / the reference.
"""

from __future__ import annotations

import json
import math

import numpy as np
import pytest

import harness as H
import synth_harness  # noqa: F401  (puts oracle/ on sys.path)
from paper_2505_11916_b200 import stats as ST

import stats_oracle as SO  # noqa: E402


def golden_cases():
    meta = json.loads((H.GOLDEN / "trace_stats.json").read_text())
    z = np.load(H.GOLDEN / "trace_stats.npz")
    for c in meta["cases"]:
        n = c["name"]
        yield c, (z[f"{n}__arrival"], z[f"{n}__input"], z[f"{n}__output"])


def assert_stats_equal(got: dict, exp: dict, name: str, corr_rtol: float = 0.0) -> None:
    assert got["num_requests"] == exp["num_requests"], name
    for k in ("duration_s", "mean_rate", "input_bucket_cv", "output_bucket_cv"):
        assert np.float64(got[k]).tobytes() == np.float64(exp[k]).tobytes(), (name, k, got[k], exp[k])
    assert [list(b) for b in got["buckets"]] == [list(b) for b in exp["buckets"]], name
    ip = {int(k): v for k, v in exp["input_percentiles"].items()}
    op = {int(k): v for k, v in exp["output_percentiles"].items()}
    assert got["input_percentiles"] == ip and got["output_percentiles"] == op, name
    if corr_rtol == 0.0:
        assert got["io_correlation"] == exp["io_correlation"], name
    else:
        assert math.isclose(got["io_correlation"], exp["io_correlation"], rel_tol=corr_rtol, abs_tol=1e-15), (
            name, got["io_correlation"], exp["io_correlation"])


def test_oracle_matches_reference_golden():
    for c, (a, i, o) in golden_cases():
        got = SO.trace_stats_arrays(a, i, o, c["bucket_s"])
        assert_stats_equal(got, c, c["name"])
        assert math.copysign(1.0, got["duration_s"]) == c["duration_sign"], c["name"]


def test_percentile_from_order_matches_numpy():
    rng = np.random.default_rng(90)
    for trial in range(400):
        n = int(rng.integers(1, 3000)) if trial % 4 else int(rng.integers(1, 12))
        v = rng.integers(1, [5, 100, 20000, 2**31 - 1][trial % 4], size=n)
        s = np.sort(v)
        for p in (50, 90, 99):
            assert ST.percentile_from_order(n, lambda k: int(s[k]), p) == int(np.percentile(v.astype(float), p))


def test_pearson_from_moments_close_to_numpy():
    for c, (a, i, o) in golden_cases():
        n = len(a)
        x = [int(v) for v in i]
        y = [int(v) for v in o]
        if n >= 2 and min(x) != max(x) and min(y) != max(y):
            r = ST.pearson_from_moments(n, sum(x), sum(y), sum(v * v for v in x), sum(v * v for v in y),
                                        sum(p * q for p, q in zip(x, y)))
        else:
            r = 0.0
        assert math.isclose(r, c["io_correlation"], rel_tol=1e-12, abs_tol=1e-15), (c["name"], r, c["io_correlation"])


def _partials_of(a, i, o, cuts) -> np.ndarray:
    """Per-chunk partials as the kernel's blocks would emit them."""
    rows = []
    for lo, hi in zip(cuts, cuts[1:]):
        p = np.zeros((), dtype=ST.PARTIAL_DTYPE)
        if hi > lo:
            p["min_arrival"], p["max_arrival"] = a[lo:hi].min(), a[lo:hi].max()
            x, y = [int(v) for v in i[lo:hi]], [int(v) for v in o[lo:hi]]
            p["count"] = hi - lo
            p["sum_x"], p["sum_y"] = sum(x), sum(y)
            for f, val in (("sxx", sum(v * v for v in x)), ("syy", sum(v * v for v in y)),
                           ("sxy", sum(u * v for u, v in zip(x, y)))):
                p[f + "_lo"], p[f + "_hi"] = val & (2**64 - 1), val >> 64
        else:
            p["min_arrival"] = p["max_arrival"] = np.nan
        rows.append(p)
    return np.array(rows, dtype=ST.PARTIAL_DTYPE)


def test_merge_of_partials():
    for c, (a, i, o) in golden_cases():
        n = len(a)
        rng = np.random.default_rng(len(c["name"]))
        cuts = sorted({0, n, *rng.integers(0, n + 1, size=7).tolist()})
        m = ST._merge(_partials_of(a, i, o, cuts))
        assert m["n"] == n
        # equal up to the sign of a zero (unobservable in TraceStats)
        assert m["first"] == min(a.tolist()) and m["last"] == max(a.tolist()), c["name"]
        assert m["sx"] == int(i.sum()) and m["sy"] == int(o.sum())


def test_bucket_limit():
    import torch

    if not torch.cuda.is_available():
        from paper_2505_11916_b200._backend import EvaluatorUnavailable

        with pytest.raises(EvaluatorUnavailable):
            ST.trace_stats([ST.TraceRequest(0, 0.0, 1, 1)])
    with pytest.raises(ValueError, match="empty"):
        ST.trace_stats([])
    with pytest.raises(ValueError, match="positive"):
        ST.trace_stats([ST.TraceRequest(0, 0.0, 1, 1)], bucket_s=0.0)
