/*
 * arrow_sim.h — C-ABI of the B200 batched evaluator for Arrow's adaptive
 * prefill/decode scheduler (arXiv 2505.11916).
 *
 * The reference path is the pure-Python discrete-event simulator `pdsim`
 * (/root/reference/pkg/src/pdsim).  It has no native code and therefore no
 * FFI of its own; this header is the boundary a maintainer would bind with
 * ctypes so that the reference's Python entry points keep their signatures
 * (see INTEGRATION.md):
 *
 *   arrow_sim_run()   replaces, per scenario, the whole of
 *                       engine.run / _Simulation.run      engine.py:259-321
 *                       (+ scheduler.py:151-335, instance.py:96-346,
 *                        pools.py:76-123, cost_model.py:73-92,
 *                        core.py:105-156 record/SLO flags)
 *                     and, per scenario, the aggregation
 *                       report.compute_metrics            report.py:55-74
 *                     so that report.run_rate_sweep (report.py:77-91) and
 *                     report.sweep_max_rate (report.py:103-109) become one
 *                     batched launch.
 *
 * All pointers are caller-owned DEVICE pointers (host pointers for the CPU
 * oracle, which shares these structs).  No allocation and no host
 * synchronisation happen inside arrow_sim_run; per-scenario failures are
 * reported through arrow_summary_t.status, launch failures through the
 * return code.  Host code maps statuses onto the reference's exceptions
 * (SimulationStallError engine.py:35-36, AssertionError engine.py:288-290,
 * RuntimeError scheduler.py:193).
 */
#ifndef ARROW_SIM_H
#define ARROW_SIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ARROW_SIM_ABI_VERSION 3

/* scheduler.py:25-28 */
enum arrow_strategy {
  ARROW_STRATEGY_SLO_AWARE = 0,
  ARROW_STRATEGY_MINIMAL_LOAD = 1,
  ARROW_STRATEGY_ROUND_ROBIN = 2
};

/* core.py:24-34 (declaration order) */
enum arrow_pool {
  ARROW_POOL_PREFILL = 0,
  ARROW_POOL_DECODE = 1,
  ARROW_POOL_P_TO_D = 2,
  ARROW_POOL_D_TO_P = 3
};

/* decision kinds, scheduler.py:104-122 */
enum arrow_decision_kind {
  ARROW_DEC_PREFILL_DISPATCH = 0,
  ARROW_DEC_DECODE_DISPATCH = 1,
  ARROW_DEC_FLIP = 2
};

/* dispatch branches, scheduler.py:151-254 */
enum arrow_branch {
  ARROW_BR_ROUND_ROBIN = 0,
  ARROW_BR_MIN_LOAD = 1,
  ARROW_BR_ALG1_T1 = 2,
  ARROW_BR_ALG1_T2 = 3,
  ARROW_BR_ALG1_FLIP = 4,
  ARROW_BR_ALG1_FALLBACK = 5,
  ARROW_BR_ALG1_DEGENERATE = 6,
  ARROW_BR_ALG2_ZERO_TRANSFER = 7,
  ARROW_BR_ALG2_T1 = 8,
  ARROW_BR_ALG2_T2 = 9,
  ARROW_BR_ALG2_FLIP = 10,
  ARROW_BR_ALG2_FALLBACK = 11,
  ARROW_BR_ALG2_FORCED_LOCAL = 12
};

/* flip triggers, scheduler.py:122,177,239,313,335 */
enum arrow_trigger {
  ARROW_TRIG_ALG1 = 0,
  ARROW_TRIG_ALG2 = 1,
  ARROW_TRIG_MONITOR_TPOT = 2,
  ARROW_TRIG_MONITOR_IDLE = 3,
  ARROW_TRIG_DRAINED = 4
};

/* per-scenario outcome */
enum arrow_status {
  ARROW_OK = 0,
  ARROW_STALLED = 1,          /* SimulationStallError raised inside the loop, engine.py:283-284 */
  ARROW_INCOMPLETE = 2,       /* heap drained with completed < n, engine.py:286-287 */
  ARROW_NOT_DRAINED = 3,      /* AssertionError, engine.py:288-290 */
  ARROW_NO_INSTANCE = 4,      /* RuntimeError, scheduler.py:192-193 */
  ARROW_ZERO_DIVISION = 5,    /* aggregate / capacity with max_tokens == 0, scheduler.py:322 */
  ARROW_BUFFER_OVERFLOW = 6,  /* a caller-sized buffer or ring was too small; re-run larger */
  ARROW_INTERNAL = 7,         /* an invariant the reference raises on was violated */
  ARROW_AUDIT_FAILED = 8      /* audit build: per-step KV / partition check failed (engine.py:279-282) */
};

/* which buffer overflowed (arrow_summary_t.overflow) */
enum arrow_overflow {
  ARROW_OVF_NONE = 0,
  ARROW_OVF_QUEUE = 1,
  ARROW_OVF_EMISSION = 2,
  ARROW_OVF_FIFO = 3,
  ARROW_OVF_DECISIONS = 4,
  ARROW_OVF_SNAPSHOTS = 5,
  ARROW_OVF_ITERLOG = 6,
  ARROW_OVF_RUNNING = 7,
  ARROW_OVF_SEQ = 8
};

/*
 * One simulation = (trace, rate scale, cluster, policy, thresholds), every
 * field resolved on the host by the reference's own rules:
 *   predictor   fit_quadratic(profile_prefill(...))   engine.py:128-131
 *   max_tokens  max_running_tokens(...)                cost_model.py:125-139
 *   thresholds  SLO defaults                           scheduler.py:75-81
 *   n_prefill   RunConfig.initial_split()              engine.py:77-83
 *   scale       native_rate(trace) / rate              report.py:85-88
 */
typedef struct arrow_scenario {
  int64_t trace_offset;     /* first request in the concatenated trace arrays */
  int32_t n_requests;
  int32_t n_instances;      /* 1..64 */
  int32_t n_prefill_init;   /* ids [0, n_prefill_init) start in PREFILL, rest in DECODE */
  int32_t strategy;         /* arrow_strategy */
  int32_t enable_flips;
  int32_t kv_capacity;      /* tokens */
  int32_t chunk_budget;
  int32_t max_batch;
  int64_t bytes_per_token;
  int64_t max_tokens;
  int64_t stall_limit;      /* engine.STALL_EVENT_LIMIT, read per call */
  double arrival_scale;     /* arrival' = arrival * scale (1.0 leaves the trace as given) */
  double true_a2, true_a1, true_a0;   /* execution prefill cost */
  double pred_a2, pred_a1, pred_a0;   /* fitted predictor (scheduler + monitor) */
  double b1, b0;                      /* decode_iter_time */
  double base_latency, bandwidth;     /* transfer_time */
  double ttft_slo, tpot_slo;
  double ttft_thr, tpot_thr;
  double theta_d, theta_busy;
  double breach_duration;
  double monitor_period;
  double window;                      /* interval_window_s */
  double min_iteration;               /* lower bound on any iteration's duration (lookahead), <= 0 if none */
} arrow_scenario_t;

/* Optional per-scenario output placement; an offset < 0 disables that output. */
typedef struct arrow_outmap {
  int64_t req_offset;         /* into req_* arrays, [req_offset, req_offset + n) */
  int64_t decision_offset;    /* into decisions */
  int64_t decision_capacity;
  int64_t snapshot_offset;    /* into snapshots, one record per (tick, instance) */
  int64_t snapshot_capacity;
  int64_t iterlog_offset;     /* into iterlog, instance i at + i * iterlog_stride */
  int64_t iterlog_stride;
  int64_t diag_offset;        /* into diag, one record per instance */
  int64_t token_offset;       /* oracle only: token_times, request r at + prefix(out)[r] */
} arrow_outmap_t;

/* report.RunSummary (report.py:31-52) plus the run's control-path digest. */
typedef struct arrow_summary {
  int32_t status;             /* arrow_status */
  int32_t overflow;           /* arrow_overflow */
  int32_t n_requests;
  int32_t n_completed;
  int32_t n_ok;               /* SLO-attaining requests */
  int32_t n_flips;
  int64_t n_events;           /* heap pops */
  int64_t n_iterations;       /* ITERATION_COMPLETE events */
  int64_t n_decisions;
  int64_t n_ticks;
  int64_t n_snapshots;        /* (tick, instance) records written */
  double stall_time;          /* time of the raising event (NaN when raised after the loop) */
  double attainment;
  double p90_ttft;
  double p90_tpot;
  double mean_ttft;
  double mean_tpot;
  double goodput;
  double span;
  uint64_t decision_hash;     /* FNV-1a over the decision stream */
  int64_t n_serial_steps;     /* evaluator: events executed one at a time */
  int64_t n_parallel_steps;   /* evaluator: lane-parallel rounds + chain bursts */
  int64_t cycles;             /* evaluator: SM clock cycles spent on this scenario */
  int64_t reserved;
} arrow_summary_t;

/* One entry of GlobalScheduler.decisions (scheduler.py:104-122). */
typedef struct arrow_decision {
  double time;
  int32_t request;            /* trace index; -1 for flips */
  int16_t instance;
  uint8_t kind;               /* arrow_decision_kind */
  uint8_t code;               /* branch, or for flips trigger | from << 3 | to << 5 */
} arrow_decision_t;

/* monitor.InstanceStats (monitor.py:19-29) at one tick. */
typedef struct arrow_snapshot {
  double time;
  double pred_delay;
  double avg_interval;        /* NaN encodes None */
  int32_t instance;
  int32_t pool;
  int32_t running_tokens;
  int32_t kv_used;
  int32_t queue_len;
  int32_t prefill_count;
  int32_t decode_count;
  int32_t reserved;
} arrow_snapshot_t;

/* Per-instance state for the SimulationStallError message (engine.py:305-316). */
typedef struct arrow_instdiag {
  double busy_until;          /* NaN encodes None */
  int32_t pool;
  int32_t kv_used;
  int32_t running;
  int32_t waiting;
  int32_t migrating;
  int32_t reserved;
} arrow_instdiag_t;

typedef struct arrow_batch {
  int32_t n_scenarios;
  int32_t flags;              /* ARROW_SIM_FORCE_*: kernel build override (0 = by batch size) */
  /* sizing (max over scenarios), used for workspace layout */
  int32_t max_requests;
  int32_t max_instances;
  int32_t queue_capacity;     /* per-instance wait/migration ring slots (<= max_requests) */
  int32_t emission_capacity;  /* per-instance token-emission ring slots */
  int32_t running_capacity;   /* per-instance running-decode slots (>= min(max_batch, chunk_budget)) */
  int32_t fifo_capacity;      /* pending PREFILL_COMPLETE slots per scenario */
  /* concatenated traces, trace index order */
  const double* arrival;
  const int32_t* input_len;
  const int32_t* output_len;
  const arrow_scenario_t* scenarios;
  const int32_t* order;       /* optional dispatch order of scenario ids (NULL = identity) */
  const arrow_outmap_t* outmap; /* optional, NULL = summaries only */
  arrow_summary_t* summaries;
  /* optional per-request outputs */
  double* req_first;          /* first token time */
  double* req_last;           /* last token time */
  int32_t* req_prefill;       /* instance | branch << 16 */
  int32_t* req_decode;        /* instance | branch << 16, -1 when output_len == 1 */
  int32_t* req_decode_iter;   /* iteration index of the decode admission, -1 when none */
  arrow_decision_t* decisions;
  arrow_snapshot_t* snapshots;
  double* iterlog;            /* completion time of every iteration, per instance */
  arrow_instdiag_t* diag;
  double* token_times;        /* oracle only */
} arrow_batch_t;

/* arrow_batch_t.flags: the latency build (unbounded registers) is chosen when
 * the batch fits in one wave of resident warps, the occupancy build otherwise;
 * these force one (same results, different speed; used by the parity tests). */
#define ARROW_SIM_FORCE_LATENCY 1
#define ARROW_SIM_FORCE_THROUGHPUT 2

/* ---- device library (libarrow_sim.so) ---- */

int arrow_sim_abi_version(void);

/* Bytes of device workspace arrow_sim_run needs for this batch's sizing. */
int arrow_sim_workspace_size(const arrow_batch_t* batch, size_t* bytes);

/* Enqueue the whole batch on `stream` (a cudaStream_t, NULL = legacy default).
 * Returns 0 on a successful launch, a cudaError_t value otherwise. */
int arrow_sim_run(const arrow_batch_t* batch, void* workspace, size_t workspace_bytes,
                  void* stream);

/* Number of resident scenario slots (warps) the persistent kernel uses. */
int arrow_sim_slots(const arrow_batch_t* batch, int* slots);

const char* arrow_sim_status_string(int status);

/* Sizes of the seven structs above, then every field offset in declaration
 * order (for binding self-checks).  Returns the number of values. */
int arrow_sim_layout(int64_t* out, int cap);

#ifdef __cplusplus
}
#endif

#endif /* ARROW_SIM_H */
