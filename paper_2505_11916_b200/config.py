"""Run configuration (mirrors RunConfig / InstanceConfig / SchedulerConfig and
the flat ``key = value`` config format of the reference).

References: InstanceConfig instance.py:33-51, Strategy/SchedulerConfig
scheduler.py:25-45, RunConfig engine.py:48-83, config keys and defaults
engine.py:328-387, parsing engine.py:390-458.  Every validation error the
reference raises is raised here, before anything reaches the device.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from pathlib import Path

from .core import SLOConfig
from .cost_model import DecodeCostParams, PrefillCostParams, TransferParams


class Strategy(Enum):
    SLO_AWARE = "slo-aware"
    MINIMAL_LOAD = "minimal-load"
    ROUND_ROBIN = "round-robin"


@dataclass(frozen=True)
class InstanceConfig:
    kv_capacity_tokens: int
    true_prefill: PrefillCostParams
    true_decode: DecodeCostParams
    transfer: TransferParams
    chunk_budget: int = 512
    max_batch_requests: int = 256

    def __post_init__(self) -> None:
        if self.chunk_budget < 1:
            raise ValueError(f"chunk_budget must be >= 1, got {self.chunk_budget}")
        if self.max_batch_requests < 1:
            raise ValueError(f"max_batch_requests must be >= 1, got {self.max_batch_requests}")
        if self.kv_capacity_tokens < self.chunk_budget:
            raise ValueError(
                f"kv_capacity_tokens {self.kv_capacity_tokens} smaller than chunk_budget {self.chunk_budget}"
            )


@dataclass(frozen=True)
class SchedulerConfig:
    strategy: Strategy = Strategy.SLO_AWARE
    ttft_threshold: float | None = None
    tpot_threshold: float | None = None
    theta_d: float = 0.5
    theta_busy: float = 0.75
    tpot_breach_duration_s: float | None = None
    enable_flips: bool = True

    def __post_init__(self) -> None:
        for name in ("theta_d", "theta_busy"):
            value = getattr(self, name)
            if not 0 < value <= 1:
                raise ValueError(f"{name} must be in (0, 1], got {value}")


@dataclass(frozen=True)
class RunConfig:
    instance_count: int
    instance: InstanceConfig
    slo: SLOConfig
    scheduler: SchedulerConfig = SchedulerConfig()
    init_prefill: int | None = None
    init_decode: int | None = None
    monitor_period_s: float = 1.0
    interval_window_s: float = 5.0
    seed: int = 0
    profile_noise: float = 0.0
    profile_points: int = 16
    max_context: int = 16384
    audit: bool = False

    def __post_init__(self) -> None:
        if self.instance_count < 1:
            raise ValueError(f"instance_count must be >= 1, got {self.instance_count}")
        if self.monitor_period_s <= 0 or self.interval_window_s <= 0:
            raise ValueError("monitor_period_s and interval_window_s must be positive")
        n_p, n_d = self.initial_split()
        if min(n_p, n_d) < 0 or n_p + n_d != self.instance_count:
            raise ValueError(f"initial split ({n_p}, {n_d}) does not partition {self.instance_count} instances")
        if self.scheduler.strategy is not Strategy.SLO_AWARE and 0 in (n_p, n_d):
            raise ValueError("static strategies need at least one instance in each pool")

    def initial_split(self) -> tuple[int, int]:
        p, d, n = self.init_prefill, self.init_decode, self.instance_count
        if p is None and d is None:
            p = (n + 1) // 2
            return p, n - p
        return (p if p is not None else n - d), (d if d is not None else n - p)


def _parse_bool(text: str) -> bool:
    return text.lower() in ("1", "true", "yes")


CONFIG_KEYS = {
    "instances": int,
    "kv_capacity_tokens": int,
    "chunk_budget": int,
    "max_batch_requests": int,
    "a2": float,
    "a1": float,
    "a0": float,
    "b1": float,
    "b0": float,
    "bytes_per_token": int,
    "bandwidth": float,
    "base_latency": float,
    "ttft_slo": float,
    "tpot_slo": float,
    "attainment_target": float,
    "strategy": str,
    "ttft_threshold": float,
    "tpot_threshold": float,
    "theta_d": float,
    "theta_busy": float,
    "tpot_breach_duration_s": float,
    "enable_flips": _parse_bool,
    "monitor_period_s": float,
    "interval_window_s": float,
    "seed": int,
    "init_prefill": int,
    "init_decode": int,
    "profile_noise": float,
    "profile_points": int,
    "max_context": int,
}

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


def parse_config_text(text: str, source: str = "<config>") -> dict:
    values = dict(DEFAULTS)
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ValueError(f"{source}:{lineno}: expected `key = value`, got {raw!r}")
        key, value = (part.strip() for part in line.split("=", 1))
        parser = CONFIG_KEYS.get(key)
        if parser is None:
            raise ValueError(f"{source}:{lineno}: unknown config key {key!r}")
        try:
            values[key] = parser(value)
        except ValueError as exc:
            raise ValueError(f"{source}:{lineno}: bad value for {key!r}: {value!r}") from exc
    return values


def config_from_values(values: dict) -> RunConfig:
    v = values
    return RunConfig(
        instance_count=v["instances"],
        instance=InstanceConfig(
            kv_capacity_tokens=v["kv_capacity_tokens"],
            true_prefill=PrefillCostParams(v["a2"], v["a1"], v["a0"]),
            true_decode=DecodeCostParams(v["b1"], v["b0"]),
            transfer=TransferParams(
                bandwidth=v["bandwidth"], base_latency=v["base_latency"], bytes_per_token=v["bytes_per_token"]
            ),
            chunk_budget=v["chunk_budget"],
            max_batch_requests=v["max_batch_requests"],
        ),
        slo=SLOConfig(ttft_slo=v["ttft_slo"], tpot_slo=v["tpot_slo"], attainment_target=v["attainment_target"]),
        scheduler=SchedulerConfig(
            strategy=Strategy(v["strategy"]),
            ttft_threshold=v.get("ttft_threshold"),
            tpot_threshold=v.get("tpot_threshold"),
            theta_d=v["theta_d"],
            theta_busy=v["theta_busy"],
            tpot_breach_duration_s=v.get("tpot_breach_duration_s"),
            enable_flips=v["enable_flips"],
        ),
        init_prefill=v.get("init_prefill"),
        init_decode=v.get("init_decode"),
        monitor_period_s=v["monitor_period_s"],
        interval_window_s=v["interval_window_s"],
        seed=v["seed"],
        profile_noise=v["profile_noise"],
        profile_points=v["profile_points"],
        max_context=v["max_context"],
    )


def load_run_config(path: str | Path) -> RunConfig:
    path = Path(path)
    return config_from_values(parse_config_text(path.read_text(), source=str(path)))


def default_run_config() -> RunConfig:
    return config_from_values(dict(DEFAULTS))
