"""B200 batched evaluator of Arrow's adaptive prefill/decode scheduler
(arXiv 2505.11916).

Drop-in for the reference simulator's Python surface (pdsim/__init__.py:10-128):
the discrete-event loop, cost model, request/instance schedulers and SLO
aggregation run as hand-written sm_100a CUDA (csrc/), one scenario per warp;
this package keeps the reference's entry points and types.
"""

from .config import (
    InstanceConfig,
    RunConfig,
    SchedulerConfig,
    Strategy,
    config_from_values,
    default_run_config,
    load_run_config,
    parse_config_text,
)
from .core import (
    Phase,
    PhaseRequest,
    PoolKind,
    RequestRecord,
    SimTime,
    SLOConfig,
    TraceRequest,
    compute_tpot,
    compute_ttft,
)
from .cost_model import (
    DecodeCostParams,
    PrefillCostParams,
    ProfilingSample,
    TransferParams,
    decode_iter_time,
    default_profile_grid,
    fit_quadratic,
    max_running_tokens,
    predict_prefill_time,
    profile_prefill,
    transfer_time,
)
from .device_traces import DeviceTrace, DeviceTraceSet, gen_synthetic_batch
from .engine import RunResult, SimulationStallError, run, scale_trace
from .monitor import InstanceStats, MonitorSnapshot
from .pools import LEGAL_EDGES
from .report import (
    RunSummary,
    compute_metrics,
    max_qualifying_rate,
    percentile_nearest_rank,
    run_rate_sweep,
    sweep_max_rate,
    write_outputs,
)
from .stats import BucketStats, TraceStats, trace_stats
from .sweep import evaluate_scenarios
from .traces import (
    BurstEpisode,
    SyntheticParams,
    bundled_bursty_trace,
    bundled_ramp_trace,
    gen_synthetic,
    load_trace,
    native_rate,
    save_trace,
)

__all__ = [name for name in dir() if not name.startswith("_")]
