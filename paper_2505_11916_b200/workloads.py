"""Named sweep workloads (BASELINE.json configs).

C1  single Arrow simulation: 4 instances (2/2), Poisson arrivals at 4 req/s,
    1 000 synthetic requests (seed 1).
C2  request-rate sweep, 32 rates (2..33 req/s) x {Arrow, static PD
    (minimal-load 4/4), PD-colocated (slo-aware, flips off, 8/0)}, 8
    instances, bundled bursty trace (2 606 requests), the rate-sweep config
    of test_acceptance.py:55-72.
C3  code-like / conversation-like traces x 8 rates (2..16 req/s) x the
    TTFT x TPOT SLO grid (8 x 5) x 3 policies, 8 instances: 1 920 runs
    (thresholds and the decode token cap derive from the SLO,
    scheduler.py:75-81, cost_model.py:125-139).
C4  pool-size x flip-threshold ablation: N in {16,24,32,48,64} x theta_d x
    theta_busy x breach x ttft_threshold x 2 rates, Arrow, 10 000 requests:
    1 080 runs.
C5  mixed-radix scenario sweep: 4 traces x 32 per-instance rates x 3
    policies x N in {4,8,16,32} x theta_d x theta_busy x breach duration.

Policies map onto the reference's strategies as SURVEY.md §0 finding 3
describes: PD-colocated = SLO_AWARE + enable_flips=False + all-prefill split.
"""

from __future__ import annotations

import dataclasses
import math

from ._compile import Scenario
from .config import RunConfig, SchedulerConfig, Strategy, default_run_config
from .cost_model import PrefillCostParams
from .traces import BurstEpisode, SyntheticParams, bundled_bursty_trace, bundled_ramp_trace, gen_synthetic, native_rate

POLICIES = ("arrow", "static-pd", "colocated")


def policy_config(base: RunConfig, policy: str, n: int) -> RunConfig:
    if policy == "arrow":
        sched, split = SchedulerConfig(strategy=Strategy.SLO_AWARE), (n // 2, n - n // 2)
    elif policy == "static-pd":
        sched, split = SchedulerConfig(strategy=Strategy.MINIMAL_LOAD), (n // 2, n - n // 2)
    elif policy == "colocated":
        sched, split = SchedulerConfig(strategy=Strategy.SLO_AWARE, enable_flips=False), (n, 0)
    else:
        raise ValueError(f"unknown policy {policy!r}")
    sched = dataclasses.replace(
        sched,
        theta_d=base.scheduler.theta_d,
        theta_busy=base.scheduler.theta_busy,
        tpot_breach_duration_s=base.scheduler.tpot_breach_duration_s,
    )
    return dataclasses.replace(base, instance_count=n, scheduler=sched, init_prefill=split[0], init_decode=split[1])


def sweep_base(n: int = 8) -> RunConfig:
    """test_acceptance.py:55-72: tight KV, cheap prefill."""
    base = default_run_config()
    inst = dataclasses.replace(base.instance, kv_capacity_tokens=3000, true_prefill=PrefillCostParams(2e-8, 2e-5, 2e-3))
    return dataclasses.replace(base, instance_count=n, instance=inst)


def c1_trace():
    return gen_synthetic(
        SyntheticParams(400.0, 4.0, math.log(420.0), 0.55, math.log(130.0), 0.5, (), 3500, 900, 1)
    )[:1000]


def c1() -> list[Scenario]:
    trace = c1_trace()
    cfg = dataclasses.replace(default_run_config(), instance_count=4, init_prefill=2, init_decode=2)
    return [Scenario(trace, cfg, native_rate(trace) / 4.0, ("c1", 4.0))]


def c2(trace=None, rates=None) -> list[Scenario]:
    trace = trace if trace is not None else bundled_bursty_trace()
    rates = rates if rates is not None else [2.0 + k for k in range(32)]
    base = sweep_base(8)
    out = []
    native = native_rate(trace)
    for policy in POLICIES:
        cfg = policy_config(base, policy, 8)
        for rate in sorted(rates):
            out.append(Scenario(trace, cfg, native / rate, (policy, rate)))
    return out


def c2_variant_trace(seed: int):
    """Bursty trace of C2 with a different generator seed (weak-scaling
    shards: rank r evaluates the C2 grid on variant r, variant 0 = C2)."""
    if seed == 0:
        return bundled_bursty_trace()
    return gen_synthetic(
        SyntheticParams(
            duration_s=360.0, base_rate=4.0, input_log_mean=math.log(420.0), input_log_sigma=0.55,
            output_log_mean=math.log(130.0), output_log_sigma=0.5,
            bursts=(BurstEpisode(50.0, 25.0, 5.0), BurstEpisode(150.0, 30.0, 4.0), BurstEpisode(260.0, 25.0, 5.0)),
            max_input=3500, max_output=900, seed=20240817 + seed,
        )
    )


def code_like_trace():
    return gen_synthetic(SyntheticParams(600.0, 4.0, math.log(1500), 0.9, math.log(40), 0.8,
                                         (BurstEpisode(60, 30, 5), BurstEpisode(240, 45, 4), BurstEpisode(450, 30, 6)),
                                         8000, 1000, 101))


def conversation_like_trace():
    return gen_synthetic(SyntheticParams(600.0, 4.0, math.log(800), 0.8, math.log(250), 0.6,
                                         (BurstEpisode(120, 120, 1.5), BurstEpisode(360, 120, 2.0)), 8000, 2000, 202))


C3_RATES = (2.0, 4.0, 6.0, 8.0, 10.0, 12.0, 14.0, 16.0)
C3_TTFT = (0.25, 0.5, 1.0, 2.0, 3.0, 5.0, 10.0, 30.0)
C3_TPOT = (0.025, 0.05, 0.075, 0.1, 0.15)


def c3(ids=None) -> list[Scenario]:
    """Scenario id -> (trace, rate, ttft slo, tpot slo, policy) in mixed radix
    2 x 8 x 8 x 5 x 3 = 1 920."""
    traces = [code_like_trace(), conversation_like_trace()]
    natives = [native_rate(t) for t in traces]
    base = default_run_config()
    total = 2 * 8 * 8 * 5 * 3
    out = []
    cache: dict = {}
    for sid in (range(total) if ids is None else ids):
        x = int(sid)
        tr, x = x % 2, x // 2
        k, x = x % 8, x // 8
        a, x = x % 8, x // 8
        b, x = x % 5, x // 5
        pol = x % 3
        key = (a, b, pol)
        cfg = cache.get(key)
        if cfg is None:
            slo = dataclasses.replace(base.slo, ttft_slo=C3_TTFT[a], tpot_slo=C3_TPOT[b])
            cfg = cache[key] = policy_config(dataclasses.replace(base, slo=slo), POLICIES[pol], 8)
        out.append(Scenario(traces[tr], cfg, natives[tr] / C3_RATES[k], sid))
    return out


def c4_trace():
    return gen_synthetic(SyntheticParams(3600.0, 4.0, math.log(420), 0.55, math.log(130), 0.5,
                                         (BurstEpisode(600, 120, 5), BurstEpisode(1800, 180, 4)), 3500, 900, 3))[:10000]


C4_N = (16, 24, 32, 48, 64)
C4_THETA_D = (0.25, 0.5, 0.75, 1.0)
C4_THETA_BUSY = (0.5, 0.75, 0.9)
C4_BREACH = (1.0, 2.0, 4.0)
C4_TTFT_FACTOR = (0.5, 0.75, 1.0)
C4_RATE_FACTOR = (1.25, 2.5)


def c4(ids=None) -> list[Scenario]:
    """Scenario id -> (N, theta_d, theta_busy, breach, ttft threshold, rate)
    in mixed radix 5 x 4 x 3 x 3 x 3 x 2 = 1 080, Arrow."""
    trace = c4_trace()
    native = native_rate(trace)
    base = default_run_config()
    total = 5 * 4 * 3 * 3 * 3 * 2
    out = []
    for sid in (range(total) if ids is None else ids):
        x = int(sid)
        ni, x = x % 5, x // 5
        td, x = x % 4, x // 4
        tb, x = x % 3, x // 3
        br, x = x % 3, x // 3
        tf, x = x % 3, x // 3
        rf = x % 2
        n = C4_N[ni]
        sched = dataclasses.replace(base.scheduler, theta_d=C4_THETA_D[td], theta_busy=C4_THETA_BUSY[tb],
                                    tpot_breach_duration_s=C4_BREACH[br],
                                    ttft_threshold=C4_TTFT_FACTOR[tf] * base.slo.ttft_slo)
        cfg = policy_config(dataclasses.replace(base, scheduler=sched), "arrow", n)
        cfg = dataclasses.replace(cfg, scheduler=dataclasses.replace(cfg.scheduler,
                                                                     ttft_threshold=sched.ttft_threshold))
        out.append(Scenario(trace, cfg, native / (C4_RATE_FACTOR[rf] * n), sid))
    return out


C5_THETA_D = (0.25, 0.5, 0.75, 1.0)
C5_THETA_BUSY = (0.5, 0.75, 0.9, 1.0)
C5_BREACH = (1.0, 2.0, 4.0, 8.0)
C5_N = (4, 8, 16, 32)


def c5(ids=None) -> list[Scenario]:
    """Scenario id -> (trace, rate k, policy, N, theta_d, theta_busy, breach)
    in mixed radix 4 x 32 x 3 x 4 x 4 x 4 x 4 = 98 304."""
    traces = [bundled_bursty_trace(), code_like_trace(), conversation_like_trace(), bundled_ramp_trace()]
    natives = [native_rate(t) for t in traces]
    base = default_run_config()
    total = 4 * 32 * 3 * 4 * 4 * 4 * 4
    ids = range(total) if ids is None else ids
    cache: dict = {}
    out = []
    for sid in ids:
        x = int(sid)
        tr, x = x % 4, x // 4
        k, x = x % 32, x // 32
        pol, x = x % 3, x // 3
        ni, x = x % 4, x // 4
        td, x = x % 4, x // 4
        tb, x = x % 4, x // 4
        br = x % 4
        n = C5_N[ni]
        key = (pol, n, td, tb, br)
        cfg = cache.get(key)
        if cfg is None:
            sched = dataclasses.replace(base.scheduler, theta_d=C5_THETA_D[td], theta_busy=C5_THETA_BUSY[tb],
                                        tpot_breach_duration_s=C5_BREACH[br])
            cfg = cache[key] = policy_config(dataclasses.replace(base, scheduler=sched), POLICIES[pol], n)
        rate = n * 0.25 * 16.0 ** (k / 31.0)
        out.append(Scenario(traces[tr], cfg, natives[tr] / rate, sid))
    return out
