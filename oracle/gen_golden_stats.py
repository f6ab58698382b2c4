"""Golden vectors for trace_stats (TEST INFRASTRUCTURE).

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden_stats.py

Runs the REAL reference ``pdsim.trace_stats`` (traces.py:202-250, imported
read-only from /root/reference/pkg/src) on the traces of ``stats_cases()``
and writes the inputs to tests/golden/trace_stats.npz and the results to
tests/golden/trace_stats.json (floats via repr, so they round-trip exactly).
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

OUT = HERE.parent / "tests" / "golden"


def stats_cases(make, synth) -> list[tuple[str, list, float]]:
    """(name, trace, bucket_s); ``make(i, arrival, in, out)`` builds a
    TraceRequest, ``synth(name)`` a catalogue trace of synth_catalogue."""
    out = []
    bursty = synth("bursty")
    out += [("bursty_60", bursty, 60.0), ("bursty_7p5", bursty, 7.5), ("bursty_0p1", bursty, 0.1)]
    out += [("code_like_10", synth("code_like"), 10.0), ("conversation_1", synth("conversation_like"), 1.0)]
    out += [("ramp_30", synth("ramp"), 30.0), ("high_rate_0p25", synth("high_rate"), 0.25)]
    out.append(("constant", [make(i, float(i), 100, 50) for i in range(300)], 60.0))     # test_traces.py:154-163
    rng = np.random.default_rng(2)
    prop = []
    for i in range(200):
        k = int(rng.integers(10, 500))
        prop.append(make(i, float(i), k, 2 * k))
    out.append(("proportional", prop, 60.0))                                          # test_traces.py:166-172
    out.append(("gaps", [make(0, 10.0, 5, 5), make(1, 130.0, 7, 5)], 60.0))           # test_traces.py:175-181
    out.append(("single", [make(0, 3.5, 17, 9)], 60.0))
    rng = np.random.default_rng(7)
    arr = np.sort(rng.uniform(0, 500, 3000))
    perm = rng.permutation(3000)
    out.append(("unsorted", [make(i, float(arr[perm[i]]), int(rng.integers(1, 4000)), int(rng.integers(1, 900)))
                             for i in range(3000)], 20.0))
    out.append(("signed_zero", [make(0, 0.0, 3, 4), make(1, -0.0, 5, 6), make(2, 0.0, 7, 8)], 60.0))
    out.append(("all_zero_time", [make(i, 0.0, 10 + i, 20 + 2 * i) for i in range(50)], 60.0))
    long_in = [make(i, 0.5 * i, int(rng.integers(1, 200_000)), int(rng.integers(16000, 70_000))) for i in range(5000)]
    out.append(("long_lengths", long_in, 100.0))
    out.append(("huge_lengths", [make(i, float(i), int(2**31 - 1 - 977 * i), int(1 + 3 * i)) for i in range(700)], 50.0))
    out.append(("big_bucket", bursty, 1e6))
    frac = [make(i, round(0.1 * i, 12), 1 + i % 7, 2 + i % 5) for i in range(400)]
    out.append(("fractional_0p1", frac, 0.1))
    out.append(("fractional_0p3", frac, 0.3))
    for k in range(4):
        r = np.random.default_rng(100 + k)
        n = int(r.integers(2, 4000))
        a = np.sort(r.exponential(1.0, n).cumsum() * float(r.uniform(0.01, 5)))
        out.append((f"random_{k}", [make(i, float(a[i]), int(r.integers(1, 20000)), int(r.integers(1, 3000)))
                                    for i in range(n)], float(r.choice([0.5, 3.0, 60.0]))))
    return out


def main() -> None:
    import pdsim
    from gen_golden_traces import catalogue  # noqa: F401  (same catalogue)
    from synth_catalogue import catalogue as cat

    kws = dict(cat())

    def synth(name):
        kw = dict(kws[name])
        kw["bursts"] = tuple(pdsim.BurstEpisode(*b) for b in kw.get("bursts", ()))
        return pdsim.gen_synthetic(pdsim.SyntheticParams(**kw))

    arrays, results = {}, []
    for name, trace, bucket in stats_cases(pdsim.TraceRequest, synth):
        s = pdsim.trace_stats(trace, bucket_s=bucket)
        arrays[f"{name}__arrival"] = np.array([r.arrival for r in trace], dtype=np.float64)
        arrays[f"{name}__input"] = np.array([r.input_len for r in trace], dtype=np.int64)
        arrays[f"{name}__output"] = np.array([r.output_len for r in trace], dtype=np.int64)
        results.append(dict(
            name=name, bucket_s=bucket, num_requests=s.num_requests, duration_s=s.duration_s,
            mean_rate=s.mean_rate, buckets=[[b.index, b.requests, b.input_tokens, b.output_tokens] for b in s.buckets],
            input_bucket_cv=s.input_bucket_cv, output_bucket_cv=s.output_bucket_cv, io_correlation=s.io_correlation,
            input_percentiles=s.input_percentiles, output_percentiles=s.output_percentiles,
            duration_sign=math.copysign(1.0, s.duration_s),
        ))
        print(f"{name:18s} n={s.num_requests:5d} buckets={len(s.buckets):6d} r={s.io_correlation:.6f}")
    np.savez_compressed(OUT / "trace_stats.npz", **arrays)
    (OUT / "trace_stats.json").write_text(json.dumps(dict(generator="oracle/gen_golden_stats.py",
                                                          numpy=np.__version__, cases=results)))
    print("wrote", OUT / "trace_stats.npz", OUT / "trace_stats.json")


if __name__ == "__main__":
    main()
