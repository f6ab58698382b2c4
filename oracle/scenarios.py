"""Parity scenario catalogue (TEST INFRASTRUCTURE).

Each entry is (name, trace_builder, config_values, scale, stall_limit,
extra).  ``config_values`` is the reference's flat key/value config
(engine.py:328-387) so the same scenario can be rebuilt by the reference
(for the golden files) and by this repo's host compiler (for the parity
tests).  Scenarios follow the reference's own tests (test_engine.py,
test_acceptance.py) and the BASELINE configs C1/C2, plus a seeded fuzz over
strategies, pool splits, thresholds and memory pressure.

Traces are built with numpy only (a duck-typed TraceRequest factory is
passed in), so this module imports neither the reference nor the product.
"""

from __future__ import annotations

import math

import numpy as np

DEFAULTS = dict(
    instances=8,
    kv_capacity_tokens=16000,
    chunk_budget=512,
    max_batch_requests=256,
    a2=1e-7,
    a1=1e-4,
    a0=5e-3,
    b1=2e-5,
    b0=5e-3,
    bytes_per_token=131072,
    bandwidth=4e11,
    base_latency=1e-4,
    ttft_slo=3.0,
    tpot_slo=0.1,
    attainment_target=0.9,
    strategy="slo-aware",
    theta_d=0.5,
    theta_busy=0.75,
    enable_flips=True,
    monitor_period_s=1.0,
    interval_window_s=5.0,
    seed=0,
    profile_noise=0.0,
    profile_points=16,
    max_context=16384,
)

# test_engine.py:38-40
ENGINE_TEST = dict(a2=2e-7, a1=1e-4, a0=2e-3, b1=1e-4, b0=4e-3)


def cfg(**kw):
    v = dict(DEFAULTS)
    v.update(kw)
    return v


def synthetic(make, duration_s, base_rate, in_mu, in_sigma, out_mu, out_sigma, bursts=(), max_input=16384,
              max_output=4096, seed=0):
    """Replays traces.gen_synthetic (traces.py:159-175) with numpy."""
    rng = np.random.default_rng(seed)
    rate_max = base_rate * max((b[2] for b in bursts), default=1.0)
    out = []
    t = 0.0
    while True:
        t += rng.exponential(1.0 / rate_max)
        if t >= duration_s:
            break
        rate = base_rate
        for start, dur, mult in bursts:
            if start <= t < start + dur:
                rate *= mult
        if rng.random() * rate_max > rate:
            continue
        i = int(min(max(round(math.exp(rng.normal(in_mu, in_sigma))), 1), max_input))
        o = int(min(max(round(math.exp(rng.normal(out_mu, out_sigma))), 1), max_output))
        out.append(make(len(out), float(t), i, o))
    return out


def bursty(make):
    return synthetic(make, 360.0, 4.0, math.log(420.0), 0.55, math.log(130.0), 0.5,
                     ((50.0, 25.0, 5.0), (150.0, 30.0, 4.0), (260.0, 25.0, 5.0)), 3500, 900, 20240817)


def ramp(make):
    return synthetic(make, 300.0, 1.0, math.log(500.0), 0.4, math.log(350.0), 0.35,
                     ((60.0, 40.0, 2.0), (100.0, 40.0, 4.0), (140.0, 40.0, 6.0), (180.0, 30.0, 3.0)), 3000, 1200, 7)


def c1_trace(make):
    return synthetic(make, 400.0, 4.0, math.log(420.0), 0.55, math.log(130.0), 0.5, (), 3500, 900, 1)[:1000]


def small_trace(make, n=60, seed=11, base_rate=3.0, duration=20.0):
    return synthetic(make, duration, base_rate, math.log(300), 0.5, math.log(60), 0.4, (), seed=seed)[:n]


def overload_trace(make):
    """test_acceptance.py:335-349"""
    reqs = []
    t = 0.0
    for _ in range(80):
        reqs.append((t, 200, 800))
        t += 0.1
    t = 5.0
    for _ in range(90):
        reqs.append((t, 3000, 2))
        t += 1.0 / 30.0
    reqs.sort(key=lambda r: r[0])
    return [make(i, a, il, ol) for i, (a, il, ol) in enumerate(reqs)]


def fcfs_trace(make, seed=42, n=80, gap=0.05):
    rng = np.random.default_rng(seed)
    arrivals = np.cumsum(rng.exponential(gap, size=n))
    lengths = rng.integers(1, 513, size=n)
    return [make(i, float(a), int(L), 1) for i, (a, L) in enumerate(zip(arrivals, lengths))]


def native_rate(trace):
    return (len(trace) - 1) / (trace[-1].arrival - trace[0].arrival)


def rate_scale(trace, rate):
    return native_rate(trace) / rate


def adaptive_vs_static(n, strategy, **kw):
    """test_acceptance.py:55-72"""
    return cfg(instances=n, kv_capacity_tokens=3000, a2=2e-8, a1=2e-5, a0=2e-3, strategy=strategy,
               init_prefill=n // 2, init_decode=n // 2, **kw)


def catalogue(make, include_slow=True):
    """List of scenario dicts: name, trace (list), values, scale, stall_limit."""
    S = []

    def add(name, trace, values, scale=1.0, stall_limit=500_000, full=False):
        S.append(dict(name=name, trace=trace, values=values, scale=scale, stall_limit=stall_limit, full=full))

    one = lambda n, a, i, o: [make(0, a, i, o)]  # noqa: E731
    # closed-form timelines, test_engine.py:92-151
    add("single_request", one(0, 0.0, 300, 4), cfg(instances=1, init_prefill=1, init_decode=0, **ENGINE_TEST), full=True)
    add("single_token", one(0, 0.0, 200, 1), cfg(instances=1, init_prefill=1, init_decode=0, **ENGINE_TEST), full=True)
    add("chunked_prefill", one(0, 0.0, 1300, 2), cfg(instances=1, init_prefill=1, init_decode=0, **ENGINE_TEST), full=True)
    add("migration_gap", one(0, 0.0, 400, 3),
        cfg(instances=2, strategy="minimal-load", init_prefill=1, init_decode=1, **ENGINE_TEST), full=True)
    add("fcfs_recurrence", fcfs_trace(make), cfg(instances=1, init_prefill=1, init_decode=0, **ENGINE_TEST), full=True)
    mon = dict(ENGINE_TEST, a2=0.0, a1=0.01, a0=0.0, b1=1e-9, b0=0.085)
    add("monitor_cadence", one(0, 0.0, 100, 100), cfg(instances=1, init_prefill=1, init_decode=0, **mon), full=True)
    add("stall_limit_zero", one(0, 0.0, 100, 4), cfg(instances=2, **ENGINE_TEST), stall_limit=0, full=True)
    # cross-run invariants, test_engine.py:214-255
    st = small_trace(make)
    add("small_arrow_2_2", st, cfg(instances=4, init_prefill=2, init_decode=2, **ENGINE_TEST), full=True)
    st120 = small_trace(make, n=120, duration=40.0)
    add("small_noflip", st120, cfg(instances=4, init_prefill=2, init_decode=2, enable_flips=False, **ENGINE_TEST),
        full=True)
    add("small_minload", st120, cfg(instances=4, strategy="minimal-load", init_prefill=2, init_decode=2, **ENGINE_TEST),
        full=True)
    # conservation suite, test_acceptance.py:249-286
    b400 = bursty(make)[:400]
    for label, strat, kv, rate in (("slo", "slo-aware", 3000, 9.0), ("minload", "minimal-load", 3000, 9.0),
                                   ("rr", "round-robin", 16000, 6.0)):
        add(f"conservation_{label}", b400,
            cfg(instances=8, init_prefill=4, init_decode=4, kv_capacity_tokens=kv, a2=2e-8, a1=2e-5, a0=2e-3,
                strategy=strat), scale=rate_scale(b400, rate), full=True)
    add("determinism_600", bursty(make)[:600], adaptive_vs_static(8, "slo-aware"), full=True)
    add("overload_flips", overload_trace(make), cfg(instances=4, init_prefill=2, init_decode=2), full=True)
    # C1 (BASELINE configs[0])
    c1 = c1_trace(make)
    add("c1_rate4", c1, cfg(instances=4, init_prefill=2, init_decode=2), scale=rate_scale(c1, 4.0), full=True)
    add("c1_rate8", c1, cfg(instances=4, init_prefill=2, init_decode=2), scale=rate_scale(c1, 8.0))
    # round-robin and degenerate splits
    add("rr_small", st120, cfg(instances=3, strategy="round-robin", init_prefill=1, init_decode=2, **ENGINE_TEST),
        full=True)
    add("colocated_small", st120, cfg(instances=4, init_prefill=4, init_decode=0, enable_flips=False, **ENGINE_TEST),
        full=True)
    add("all_decode_start", st120, cfg(instances=3, init_prefill=0, init_decode=3, **ENGINE_TEST), full=True)
    # memory pressure and caps
    add("tight_kv", st120, cfg(instances=4, kv_capacity_tokens=1200, chunk_budget=128, **ENGINE_TEST),
        scale=0.5, full=True)
    add("decode_cap", st120, cfg(instances=2, max_batch_requests=3, chunk_budget=64, init_prefill=1, init_decode=1,
                                 kv_capacity_tokens=4000, **ENGINE_TEST), scale=0.25, full=True)
    # stalls (small watchdog so the reference finishes quickly)
    b = bursty(make)
    if include_slow:
        add("c2_arrow_r10", b, adaptive_vs_static(8, "slo-aware"), scale=rate_scale(b, 10.0))
        add("c2_static_r10", b, adaptive_vs_static(8, "minimal-load"), scale=rate_scale(b, 10.0))
        add("c2_coloc_r10", b, adaptive_vs_static(8, "slo-aware", enable_flips=False) | dict(init_prefill=8, init_decode=0),
            scale=rate_scale(b, 10.0))
        add("c2_arrow_r32_stall", b, adaptive_vs_static(8, "slo-aware"), scale=rate_scale(b, 32.0), stall_limit=20000)
        add("c2_coloc_r20_stall", b, adaptive_vs_static(8, "slo-aware", enable_flips=False) | dict(init_prefill=8, init_decode=0),
            scale=rate_scale(b, 20.0), stall_limit=20000)
        r = ramp(make)
        add("ramp_minload", r, cfg(instances=8, init_prefill=4, init_decode=4, strategy="minimal-load"), scale=1.0 / 8.0,
            full=True)
    # seeded fuzz
    rng = np.random.default_rng(20260101)
    for k in range(40):
        N = int(rng.integers(1, 13))
        strat = ["slo-aware", "slo-aware", "minimal-load", "round-robin"][int(rng.integers(0, 4))]
        if strat != "slo-aware" and N < 2:
            N = 2
        n_p = int(rng.integers(1 if strat != "slo-aware" else 0, N if strat != "slo-aware" else N + 1))
        v = cfg(
            instances=N,
            init_prefill=n_p,
            init_decode=N - n_p,
            strategy=strat,
            enable_flips=bool(rng.integers(0, 4) > 0),
            kv_capacity_tokens=int(rng.choice([1500, 3000, 6000, 16000])),
            chunk_budget=int(rng.choice([128, 256, 512])),
            max_batch_requests=int(rng.choice([4, 16, 256])),
            theta_d=float(rng.choice([0.25, 0.5, 1.0])),
            theta_busy=float(rng.choice([0.3, 0.75, 1.0])),
            tpot_breach_duration_s=float(rng.choice([1.0, 2.0, 4.0])),
            ttft_slo=float(rng.choice([0.5, 1.0, 3.0])),
            tpot_slo=float(rng.choice([0.03, 0.1])),
            a2=2e-8, a1=2e-5, a0=2e-3,
            seed=int(rng.integers(0, 3)),
            profile_noise=float(rng.choice([0.0, 0.0, 0.02])),
        )
        if rng.integers(0, 2):
            v["ttft_threshold"] = float(rng.choice([0.25, 1.0, 2.0]))
        n_req = int(rng.integers(20, 260))
        cap = min(1400, v["kv_capacity_tokens"] // 2) if k % 10 else 1400   # every 10th: may fail validation
        tr = synthetic(make, 60.0, 3.0, math.log(float(rng.choice([150, 400, 900]))), 0.6,
                       math.log(float(rng.choice([20, 80, 200]))), 0.6, ((10.0, 10.0, 3.0),), cap, cap,
                       int(rng.integers(0, 10_000)))[:n_req]
        if len(tr) < 2:
            continue
        rate = float(rng.choice([1.0, 3.0, 6.0, 12.0])) * max(N, 1) / 4
        add(f"fuzz_{k:02d}", tr, v, scale=rate_scale(tr, rate), stall_limit=20000, full=k % 3 == 0)
    return S


# ---------------------------------------------------------------------------
# BASELINE configs C3, C4, C5 and the burst-merge tie case.
# Generated into tests/golden/ with GOLDEN_SET=r2 (oracle/gen_golden.py).

def code_like(make):
    """C3 code-like trace: 3 955 requests."""
    return synthetic(make, 600.0, 4.0, math.log(1500.0), 0.9, math.log(40.0), 0.8,
                     ((60.0, 30.0, 5.0), (240.0, 45.0, 4.0), (450.0, 30.0, 6.0)), 8000, 1000, 101)


def conversation_like(make):
    """C3 conversation-like trace: 3 133 requests."""
    return synthetic(make, 600.0, 4.0, math.log(800.0), 0.8, math.log(250.0), 0.6,
                     ((120.0, 120.0, 1.5), (360.0, 120.0, 2.0)), 8000, 2000, 202)


def c4_trace(make):
    """C4 trace: 10 000 requests."""
    return synthetic(make, 3600.0, 4.0, math.log(420.0), 0.55, math.log(130.0), 0.5,
                     ((600.0, 120.0, 5.0), (1800.0, 180.0, 4.0)), 3500, 900, 3)[:10000]


def policy_values(policy, n, **kw):
    """Arrow / static PD / PD-colocated as flat config values
    (paper_2505_11916_b200/workloads.py:policy_config, restated)."""
    if policy == "arrow":
        v = cfg(instances=n, strategy="slo-aware", init_prefill=n // 2, init_decode=n - n // 2)
    elif policy == "static-pd":
        v = cfg(instances=n, strategy="minimal-load", init_prefill=n // 2, init_decode=n - n // 2)
    elif policy == "colocated":
        v = cfg(instances=n, strategy="slo-aware", enable_flips=False, init_prefill=n, init_decode=0)
    else:
        raise ValueError(policy)
    v.update(kw)
    return v


C3_POINTS = (  # (ttft_slo, tpot_slo, rate): six points of the 8 x 5 SLO grid, rates 2..16
    (0.25, 0.025, 4.0), (0.5, 0.05, 8.0), (1.0, 0.075, 12.0), (2.0, 0.1, 16.0), (5.0, 0.15, 6.0), (30.0, 0.025, 10.0),
)

C4_POINTS = (  # (N, theta_d, theta_busy, breach, ttft_threshold factor, rate factor)
    (16, 0.25, 0.5, 1.0, 0.5, 1.25), (16, 1.0, 0.9, 4.0, 1.0, 2.5), (24, 0.5, 0.75, 2.0, 0.75, 2.5),
    (32, 0.25, 0.9, 4.0, 1.0, 1.25), (32, 1.0, 0.5, 1.0, 0.5, 2.5), (48, 0.75, 0.75, 2.0, 0.75, 1.25),
    (48, 0.25, 0.5, 4.0, 0.5, 2.5), (64, 1.0, 0.9, 1.0, 1.0, 2.5), (64, 0.5, 0.5, 2.0, 0.75, 1.25),
)

C5_RADIX = (4, 32, 3, 4, 4, 4, 4)  # trace, rate k, policy, N, theta_d, theta_busy, breach
C5_POLICIES = ("arrow", "static-pd", "colocated")
C5_N = (4, 8, 16, 32)
C5_THETA_D = (0.25, 0.5, 0.75, 1.0)
C5_THETA_BUSY = (0.5, 0.75, 0.9, 1.0)
C5_BREACH = (1.0, 2.0, 4.0, 8.0)


def c5_digits(sid):
    out = []
    for r in C5_RADIX:
        out.append(sid % r)
        sid //= r
    return out


def c5_id(tr, k, pol, ni, td, tb, br):
    sid = 0
    for d, r in zip(reversed((tr, k, pol, ni, td, tb, br)), reversed(C5_RADIX)):
        sid = sid * r + d
    return sid


def c5_stratified_ids(count=32, seed=55):
    """Every trace, policy and N appear; rate and threshold digits seeded."""
    rng = np.random.default_rng(seed)
    ids = []
    for j in range(count):
        tr, pol, ni = j % 4, j % 3, (j // 4) % 4
        k = int(rng.integers(0, 32))
        td, tb, br = (int(x) for x in rng.integers(0, 4, size=3))
        ids.append(c5_id(tr, k, pol, ni, td, tb, br))
    return ids


def c5_scenario(make, sid, traces=None):
    """Scenario id -> (trace, config values, scale), SURVEY.md §8(d) C5."""
    tr, k, pol, ni, td, tb, br = c5_digits(sid)
    if traces is None:
        traces = [bursty(make), code_like(make), conversation_like(make), ramp(make)]
    trace = traces[tr]
    n = C5_N[ni]
    v = policy_values(C5_POLICIES[pol], n, theta_d=C5_THETA_D[td], theta_busy=C5_THETA_BUSY[tb],
                      tpot_breach_duration_s=C5_BREACH[br])
    rate = n * 0.25 * 16.0 ** (k / 31.0)
    return trace, v, rate_scale(trace, rate)


def tie_lockstep_trace(make, t_arrive):
    """Burst-merge tie case.  Two PD-colocated instances get identical
    requests at t=0 and decode them in lockstep: their decode-only iteration
    chains run as chain bursts whose final pending completions fall at exactly
    the same time, so the burst merge's equal-time fallback assigns their
    sequence numbers.  Two identical short prompts arriving at t_arrive (one
    per instance) join those instances' next batches; both prefills finish
    in the same iteration on both instances, and the two PREFILL_COMPLETE
    events -- and so the two decode_dispatch records -- come out in the order
    of the tied sequence numbers.  A merge that reversed equal-time finals
    logs request 3 before request 2 (tests/test_emulated_kernel.py runs that
    mutant)."""
    reqs = [(0.0, 100, 200), (0.0, 100, 200), (t_arrive, 50, 5), (t_arrive, 50, 5)]
    return [make(i, a, il, ol) for i, (a, il, ol) in enumerate(reqs)]


TIE_ARRIVALS = (0.503, 0.52, 0.53, 0.71, 0.8)


def catalogue_r2(make, c5_count=32, which=("c3", "c4", "c5", "tie")):
    S = []

    def add(name, trace, values, scale=1.0, stall_limit=500_000, full=False):
        S.append(dict(name=name, trace=trace, values=values, scale=scale, stall_limit=stall_limit, full=full))

    if "c3" in which:
        for tname, tr in (("code", code_like(make)), ("chat", conversation_like(make))):
            for pol in C5_POLICIES:
                for p, (ttft, tpot, rate) in enumerate(C3_POINTS):
                    add(f"c3_{tname}_{pol}_{p}", tr, policy_values(pol, 8, ttft_slo=ttft, tpot_slo=tpot),
                        scale=rate_scale(tr, rate))
    if "c4" in which:
        tr = c4_trace(make)
        for p, (n, td, tb, br, tf, rf) in enumerate(C4_POINTS):
            v = policy_values("arrow", n, theta_d=td, theta_busy=tb, tpot_breach_duration_s=br,
                              ttft_threshold=tf * DEFAULTS["ttft_slo"])
            add(f"c4_{p}_n{n}", tr, v, scale=rate_scale(tr, rf * n))
    if "c5" in which:
        traces = [bursty(make), code_like(make), conversation_like(make), ramp(make)]
        for sid in c5_stratified_ids(c5_count):
            tr, v, sc = c5_scenario(make, sid, traces)
            add(f"c5_{sid:05d}", tr, v, scale=sc)
    if "adv" in which:
        # Adversarial predictors for the delay-interval bound (sim_core.cuh:
        # delay_interval): heavy profiling noise makes the fitted a2 / a1 / a0
        # negative (e.g. a0 = -0.15 s, a2 < 0), so predicted prefill terms of
        # the delay fold have mixed signs and cancel.
        tr = bursty(make)[:300]
        for k, (noise, seed) in enumerate([(1.0, 1), (1.0, 2), (1.0, 3), (3.0, 0), (3.0, 1), (3.0, 2), (3.0, 3),
                                           (10.0, 5)]):
            strat = "minimal-load" if k % 4 == 3 else "slo-aware"
            v = cfg(instances=4 + k % 4, init_prefill=2 + k % 2, init_decode=2 + k % 4 - k % 2, strategy=strat,
                    profile_noise=noise, seed=seed, kv_capacity_tokens=3000, a2=2e-8, a1=2e-5, a0=2e-3)
            add(f"adv_delay_{k}", tr, v, scale=rate_scale(tr, 6.0 + 2 * k), full=k % 2 == 0)
    if "stallchunk" in which:
        # Long prompts in small chunks: runs of token-less prefill iterations
        # that only advance the stall counter (engine.py:268).  With small
        # watchdog limits the reference raises mid-prefill, so the exact
        # event at which the counter crosses the limit is pinned.
        for k, limit in enumerate((130, 150, 200, 257, 300, 400, 1000)):
            n = 2 + k % 3
            reqs = [make(i, 0.05 * i, 6000 - 500 * (i % 4), 3 + i % 5) for i in range(6 + k)]
            v = cfg(instances=n, init_prefill=n - 1, init_decode=1, chunk_budget=32 + 16 * (k % 3),
                    kv_capacity_tokens=16000, **ENGINE_TEST)
            add(f"stallchunk_{k}", reqs, v, stall_limit=limit, full=True)
        for k, (limit, n_p) in enumerate(((300, 2), (400, 2), (500, 3), (700, 3), (333, 1))):
            reqs = [make(i, 0.01 * i, 8000 - 7 * i, 2 + i % 3) for i in range(8)]
            v = cfg(instances=n_p + 1, init_prefill=n_p, init_decode=1, chunk_budget=32, kv_capacity_tokens=40000,
                    **ENGINE_TEST)
            add(f"stallchunk_long_{k}", reqs, v, stall_limit=limit, full=True)
    if "tie" in which:
        v = cfg(instances=2, init_prefill=2, init_decode=0, enable_flips=False, **ENGINE_TEST)
        for t in TIE_ARRIVALS:
            add(f"tie_lockstep_{int(round(t * 1000)):04d}", tie_lockstep_trace(make, t), v, full=True)
    return S


# Whole-sweep restatements by scenario id (paper_2505_11916_b200/workloads.py
# c3 / c4, restated with flat reference config values) for the digest
# fixtures of oracle/gen_golden_digest.py.
C3_RATES = (2.0, 4.0, 6.0, 8.0, 10.0, 12.0, 14.0, 16.0)
C3_TTFT = (0.25, 0.5, 1.0, 2.0, 3.0, 5.0, 10.0, 30.0)
C3_TPOT = (0.025, 0.05, 0.075, 0.1, 0.15)
C4_N = (16, 24, 32, 48, 64)
C4_THETA_D = (0.25, 0.5, 0.75, 1.0)
C4_THETA_BUSY = (0.5, 0.75, 0.9)
C4_BREACH = (1.0, 2.0, 4.0)
C4_TTFT_FACTOR = (0.5, 0.75, 1.0)
C4_RATE_FACTOR = (1.25, 2.5)


def c3_scenario(make, sid, traces=None):
    """C3 id -> mixed radix (trace 2, rate 8, ttft 8, tpot 5, policy 3)."""
    x = int(sid)
    tr, x = x % 2, x // 2
    k, x = x % 8, x // 8
    a, x = x % 8, x // 8
    b, x = x % 5, x // 5
    pol = x % 3
    if traces is None:
        traces = [code_like(make), conversation_like(make)]
    trace = traces[tr]
    v = policy_values(C5_POLICIES[pol], 8, ttft_slo=C3_TTFT[a], tpot_slo=C3_TPOT[b])
    return trace, v, rate_scale(trace, C3_RATES[k])


def c4_scenario(make, sid, trace=None):
    """C4 id -> mixed radix (N 5, theta_d 4, theta_busy 3, breach 3, ttft factor 3, rate 2), Arrow."""
    x = int(sid)
    ni, x = x % 5, x // 5
    td, x = x % 4, x // 4
    tb, x = x % 3, x // 3
    br, x = x % 3, x // 3
    tf, x = x % 3, x // 3
    rf = x % 2
    n = C4_N[ni]
    if trace is None:
        trace = c4_trace(make)
    v = policy_values("arrow", n, theta_d=C4_THETA_D[td], theta_busy=C4_THETA_BUSY[tb],
                      tpot_breach_duration_s=C4_BREACH[br], ttft_threshold=C4_TTFT_FACTOR[tf] * DEFAULTS["ttft_slo"])
    return trace, v, rate_scale(trace, C4_RATE_FACTOR[rf] * n)
