"""numpy mirrors of the C structs in include/arrow_sim.h.

Arrays of these dtypes are the buffers handed across the C-ABI (host arrays
for the CPU oracle, torch device tensors viewed as raw bytes for the CUDA
library).  ``align=True`` gives the natural C layout; tests/test_abi.py
checks every size and offset against the compiled library.
"""

from __future__ import annotations

import ctypes

import numpy as np

ABI_VERSION = 3

# enums (include/arrow_sim.h)
STRATEGY_CODES = {"slo-aware": 0, "minimal-load": 1, "round-robin": 2}
POOL_NAMES = ("prefill", "decode", "p_to_d", "d_to_p")
DEC_PREFILL, DEC_DECODE, DEC_FLIP = 0, 1, 2
DECISION_KIND_NAMES = ("prefill_dispatch", "decode_dispatch", "flip")
BRANCH_NAMES = (
    "round-robin",
    "min-load",
    "alg1:t1",
    "alg1:t2",
    "alg1:flip",
    "alg1:fallback",
    "alg1:degenerate",
    "alg2:zero-transfer",
    "alg2:t1",
    "alg2:t2",
    "alg2:flip",
    "alg2:fallback",
    "alg2:forced-local",
)
TRIGGER_NAMES = ("alg1", "alg2", "monitor:tpot", "monitor:idle", "drained")

OK, STALLED, INCOMPLETE, NOT_DRAINED, NO_INSTANCE, ZERO_DIVISION, BUFFER_OVERFLOW, INTERNAL, AUDIT_FAILED = range(9)
STATUS_NAMES = (
    "ok",
    "stalled",
    "incomplete",
    "not-drained",
    "no-instance",
    "zero-division",
    "buffer-overflow",
    "internal",
    "audit-failed",
)
OVERFLOW_NAMES = ("none", "queue", "emission", "fifo", "decisions", "snapshots", "iterlog", "running", "seq")

SCENARIO_DTYPE = np.dtype(
    [
        ("trace_offset", np.int64),
        ("n_requests", np.int32),
        ("n_instances", np.int32),
        ("n_prefill_init", np.int32),
        ("strategy", np.int32),
        ("enable_flips", np.int32),
        ("kv_capacity", np.int32),
        ("chunk_budget", np.int32),
        ("max_batch", np.int32),
        ("bytes_per_token", np.int64),
        ("max_tokens", np.int64),
        ("stall_limit", np.int64),
        ("arrival_scale", np.float64),
        ("true_a2", np.float64),
        ("true_a1", np.float64),
        ("true_a0", np.float64),
        ("pred_a2", np.float64),
        ("pred_a1", np.float64),
        ("pred_a0", np.float64),
        ("b1", np.float64),
        ("b0", np.float64),
        ("base_latency", np.float64),
        ("bandwidth", np.float64),
        ("ttft_slo", np.float64),
        ("tpot_slo", np.float64),
        ("ttft_thr", np.float64),
        ("tpot_thr", np.float64),
        ("theta_d", np.float64),
        ("theta_busy", np.float64),
        ("breach_duration", np.float64),
        ("monitor_period", np.float64),
        ("window", np.float64),
        ("min_iteration", np.float64),
    ],
    align=True,
)

OUTMAP_DTYPE = np.dtype(
    [
        ("req_offset", np.int64),
        ("decision_offset", np.int64),
        ("decision_capacity", np.int64),
        ("snapshot_offset", np.int64),
        ("snapshot_capacity", np.int64),
        ("iterlog_offset", np.int64),
        ("iterlog_stride", np.int64),
        ("diag_offset", np.int64),
        ("token_offset", np.int64),
    ],
    align=True,
)

SUMMARY_DTYPE = np.dtype(
    [
        ("status", np.int32),
        ("overflow", np.int32),
        ("n_requests", np.int32),
        ("n_completed", np.int32),
        ("n_ok", np.int32),
        ("n_flips", np.int32),
        ("n_events", np.int64),
        ("n_iterations", np.int64),
        ("n_decisions", np.int64),
        ("n_ticks", np.int64),
        ("n_snapshots", np.int64),
        ("stall_time", np.float64),
        ("attainment", np.float64),
        ("p90_ttft", np.float64),
        ("p90_tpot", np.float64),
        ("mean_ttft", np.float64),
        ("mean_tpot", np.float64),
        ("goodput", np.float64),
        ("span", np.float64),
        ("decision_hash", np.uint64),
        ("n_serial_steps", np.int64),
        ("n_parallel_steps", np.int64),
        ("cycles", np.int64),
        ("reserved", np.int64),
    ],
    align=True,
)

DECISION_DTYPE = np.dtype(
    [
        ("time", np.float64),
        ("request", np.int32),
        ("instance", np.int16),
        ("kind", np.uint8),
        ("code", np.uint8),
    ],
    align=True,
)

SNAPSHOT_DTYPE = np.dtype(
    [
        ("time", np.float64),
        ("pred_delay", np.float64),
        ("avg_interval", np.float64),
        ("instance", np.int32),
        ("pool", np.int32),
        ("running_tokens", np.int32),
        ("kv_used", np.int32),
        ("queue_len", np.int32),
        ("prefill_count", np.int32),
        ("decode_count", np.int32),
        ("reserved", np.int32),
    ],
    align=True,
)

INSTDIAG_DTYPE = np.dtype(
    [
        ("busy_until", np.float64),
        ("pool", np.int32),
        ("kv_used", np.int32),
        ("running", np.int32),
        ("waiting", np.int32),
        ("migrating", np.int32),
        ("reserved", np.int32),
    ],
    align=True,
)


class Batch(ctypes.Structure):
    """arrow_batch_t: sizing + raw pointers (host or device)."""

    _fields_ = [
        ("n_scenarios", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("max_requests", ctypes.c_int32),
        ("max_instances", ctypes.c_int32),
        ("queue_capacity", ctypes.c_int32),
        ("emission_capacity", ctypes.c_int32),
        ("running_capacity", ctypes.c_int32),
        ("fifo_capacity", ctypes.c_int32),
        ("arrival", ctypes.c_void_p),
        ("input_len", ctypes.c_void_p),
        ("output_len", ctypes.c_void_p),
        ("scenarios", ctypes.c_void_p),
        ("order", ctypes.c_void_p),
        ("outmap", ctypes.c_void_p),
        ("summaries", ctypes.c_void_p),
        ("req_first", ctypes.c_void_p),
        ("req_last", ctypes.c_void_p),
        ("req_prefill", ctypes.c_void_p),
        ("req_decode", ctypes.c_void_p),
        ("req_decode_iter", ctypes.c_void_p),
        ("decisions", ctypes.c_void_p),
        ("snapshots", ctypes.c_void_p),
        ("iterlog", ctypes.c_void_p),
        ("diag", ctypes.c_void_p),
        ("token_times", ctypes.c_void_p),
    ]


POINTER_FIELDS = [name for name, typ in Batch._fields_ if typ is ctypes.c_void_p]

STRUCT_SIZES = {
    "scenario": SCENARIO_DTYPE.itemsize,
    "outmap": OUTMAP_DTYPE.itemsize,
    "summary": SUMMARY_DTYPE.itemsize,
    "decision": DECISION_DTYPE.itemsize,
    "snapshot": SNAPSHOT_DTYPE.itemsize,
    "instdiag": INSTDIAG_DTYPE.itemsize,
    "batch": ctypes.sizeof(Batch),
}


def fnv_decision_hash(decisions: np.ndarray) -> int:
    """FNV-1a over (time bits, packed kind/code/instance/request) per decision;
    the same digest the CUDA kernel and the oracle compute."""
    h = 14695981039346656037
    mask = (1 << 64) - 1
    prime = 1099511628211
    times = decisions["time"].view(np.uint64)
    for k in range(len(decisions)):
        w1 = int(times[k])
        w2 = (
            int(decisions["kind"][k])
            | (int(decisions["code"][k]) << 8)
            | ((int(decisions["instance"][k]) & 0xFFFF) << 16)
            | ((int(decisions["request"][k]) & 0xFFFFFFFF) << 32)
        )
        h = ((h ^ w1) * prime) & mask
        h = ((h ^ w2) * prime) & mask
    return h


# ---- include/arrow_traces.h (device workload generator) ----

SYNTH_MAX_BURSTS = 16
SYNTH_MAX_SEED_WORDS = 8
SYNTH_OK, SYNTH_CAPACITY, SYNTH_OVERFLOW = range(3)

SYNTH_DTYPE = np.dtype(
    [
        ("duration_s", np.float64),
        ("base_rate", np.float64),
        ("rate_max", np.float64),
        ("gap_scale", np.float64),
        ("input_log_mean", np.float64),
        ("input_log_sigma", np.float64),
        ("output_log_mean", np.float64),
        ("output_log_sigma", np.float64),
        ("max_input", np.int64),
        ("max_output", np.int64),
        ("n_bursts", np.int32),
        ("n_seed_words", np.int32),
        ("seed_words", np.uint32, (SYNTH_MAX_SEED_WORDS,)),
        ("burst_start", np.float64, (SYNTH_MAX_BURSTS,)),
        ("burst_duration", np.float64, (SYNTH_MAX_BURSTS,)),
        ("burst_multiplier", np.float64, (SYNTH_MAX_BURSTS,)),
        ("out_offset", np.int64),
        ("capacity", np.int64),
    ],
    align=True,
)

SYNTH_RESULT_DTYPE = np.dtype(
    [
        ("count", np.int64),
        ("status", np.int32),
        ("reserved", np.int32),
        ("first_arrival", np.float64),
        ("last_arrival", np.float64),
        ("max_kv", np.int64),
        ("sum_input", np.int64),
        ("sum_output", np.int64),
    ],
    align=True,
)
