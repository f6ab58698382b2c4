"""Synthetic-workload parity catalogue (TEST INFRASTRUCTURE).

Parameter sets for the device generator's golden vectors
(oracle/gen_golden_traces.py runs the real ``pdsim.gen_synthetic`` on them)
and for the CPU/GPU parity tests.  Each entry is a dict of
``SyntheticParams`` keyword arguments with bursts as (start, duration,
multiplier) tuples, so it builds both the reference's and this repo's
dataclasses.  Covers the reference's bundled workloads (traces.py:264-309),
SURVEY.md's C3/C4 generators, and the edge cases of traces.py:146-175:
overlapping and out-of-range bursts, multipliers below 1 (rate_max below
the base rate), zero duration, zero / huge log-sigma (clamping at 1 and at
max_len), max_len = 1, and seeds of 1..7 uint32 words.
"""

from __future__ import annotations

import math

L = math.log


def catalogue() -> list[tuple[str, dict]]:
    bursty = dict(duration_s=360.0, base_rate=4.0, input_log_mean=L(420.0), input_log_sigma=0.55,
                  output_log_mean=L(130.0), output_log_sigma=0.5,
                  bursts=((50.0, 25.0, 5.0), (150.0, 30.0, 4.0), (260.0, 25.0, 5.0)),
                  max_input=3500, max_output=900, seed=20240817)
    ramp = dict(duration_s=300.0, base_rate=1.0, input_log_mean=L(500.0), input_log_sigma=0.4,
                output_log_mean=L(350.0), output_log_sigma=0.35,
                bursts=((60.0, 40.0, 2.0), (100.0, 40.0, 4.0), (140.0, 40.0, 6.0), (180.0, 30.0, 3.0)),
                max_input=3000, max_output=1200, seed=7)
    code = dict(duration_s=600.0, base_rate=4.0, input_log_mean=L(1500), input_log_sigma=0.9,
                output_log_mean=L(40), output_log_sigma=0.8,
                bursts=((60, 30, 5), (240, 45, 4), (450, 30, 6)), max_input=8000, max_output=1000, seed=101)
    conv = dict(duration_s=600.0, base_rate=4.0, input_log_mean=L(800), input_log_sigma=0.8,
                output_log_mean=L(250), output_log_sigma=0.6,
                bursts=((120, 120, 1.5), (360, 120, 2.0)), max_input=8000, max_output=2000, seed=202)
    small = dict(duration_s=120.0, base_rate=3.0, input_log_mean=L(300), input_log_sigma=0.5,
                 output_log_mean=L(60), output_log_sigma=0.4, seed=11)
    out = [
        ("bursty", bursty),
        ("ramp", ramp),
        ("code_like", code),
        ("conversation_like", conv),
        ("small", small),
        ("seed0", dict(small, seed=0)),
        ("seed_2w", dict(small, seed=2**40 + 12345)),
        ("seed_3w", dict(small, seed=2**70 + 99)),
        ("seed_7w", dict(small, seed=2**200 + 3)),
        ("seed_u32max", dict(small, seed=2**32 - 1)),
        ("overlap", dict(small, bursts=((10.0, 50.0, 3.0), (30.0, 50.0, 2.0), (40.0, 5.0, 0.5)), seed=5)),
        ("mult_below_one", dict(small, bursts=((20.0, 40.0, 0.25), (70.0, 10.0, 0.5)), seed=6)),
        ("burst_outside", dict(small, bursts=((500.0, 10.0, 8.0), (-50.0, 60.0, 2.0)), seed=8)),
        ("zero_duration", dict(small, duration_s=0.0, seed=9)),
        ("sigma_zero", dict(small, input_log_sigma=0.0, output_log_sigma=0.0, seed=10)),
        ("sigma_huge", dict(small, input_log_sigma=6.0, output_log_sigma=5.0, max_input=20000,
                            max_output=3000, seed=12)),
        ("tiny_means", dict(small, input_log_mean=L(1.2), output_log_mean=L(0.7), seed=13)),
        ("max_len_one", dict(small, max_input=1, max_output=1, seed=14)),
        ("high_rate", dict(small, duration_s=20.0, base_rate=200.0, bursts=((5.0, 5.0, 3.0),), seed=15)),
        ("many_bursts", dict(small, duration_s=200.0,
                             bursts=tuple((8.0 * k, 4.0, 1.0 + (k % 5)) for k in range(16)), seed=16)),
    ]
    for k in range(8):
        out.append((f"bursty_seed{k}", dict(bursty, duration_s=120.0, seed=1000 + 7919 * k)))
    return out
