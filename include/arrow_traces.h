/*
 * arrow_traces.h — C-ABI of the device workload generator (§8(f) rank 3).
 *
 * Replaces, per trace, the reference's synthetic workload generator
 *     pdsim.traces.gen_synthetic(SyntheticParams)        traces.py:159-175
 * (thinned Poisson arrivals with burst episodes, log-normal lengths drawn
 * from numpy's default_rng(seed)), bit for bit: same PCG64 stream, same
 * ziggurat samplers, same float operations.  One launch generates a whole
 * batch of traces (one per (params, seed)) straight into device memory,
 * where the evaluator (arrow_sim.h) consumes them without a host round trip.
 *
 * The reference has no FFI (pure Python); the binding a maintainer would add
 * is the ctypes stub in INTEGRATION.md.  All pointers are caller-owned device
 * pointers; no allocation, no host synchronisation.
 */
#ifndef ARROW_TRACES_H
#define ARROW_TRACES_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ARROW_SYNTH_MAX_BURSTS 16
#define ARROW_SYNTH_MAX_SEED_WORDS 8

/* SyntheticParams (traces.py:122-143) with every Python-side derived value
 * resolved on the host by the reference's own expressions:
 *   rate_max  = base_rate * max(multipliers, default=1.0)     traces.py:162
 *   gap_scale = 1.0 / rate_max                                  traces.py:166
 *   seed      -> little-endian uint32 words (SeedSequence entropy). */
typedef struct arrow_synth {
  double duration_s;
  double base_rate;
  double rate_max;
  double gap_scale;
  double input_log_mean, input_log_sigma;
  double output_log_mean, output_log_sigma;
  int64_t max_input;
  int64_t max_output;
  int32_t n_bursts;                       /* <= ARROW_SYNTH_MAX_BURSTS, declaration order */
  int32_t n_seed_words;                   /* 1..ARROW_SYNTH_MAX_SEED_WORDS */
  uint32_t seed_words[ARROW_SYNTH_MAX_SEED_WORDS];
  double burst_start[ARROW_SYNTH_MAX_BURSTS];
  double burst_duration[ARROW_SYNTH_MAX_BURSTS];
  double burst_multiplier[ARROW_SYNTH_MAX_BURSTS];
  int64_t out_offset;                     /* first slot of this trace in the output arrays */
  int64_t capacity;                       /* slots available at out_offset */
} arrow_synth_t;

enum arrow_synth_status {
  ARROW_SYNTH_OK = 0,
  ARROW_SYNTH_CAPACITY = 1,   /* more requests than capacity; count holds the true total */
  ARROW_SYNTH_OVERFLOW = 2    /* math.exp overflowed (OverflowError in the reference) */
};

/* Per-trace result: what the scenario compiler needs without downloading
 * the trace (native_rate traces.py:253-261, _validate_trace engine.py:101-115). */
typedef struct arrow_synth_result {
  int64_t count;              /* requests generated (len(trace)) */
  int32_t status;             /* arrow_synth_status */
  int32_t reserved;
  double first_arrival;       /* trace[0].arrival  (NaN if empty) */
  double last_arrival;        /* trace[-1].arrival (NaN if empty) */
  int64_t max_kv;             /* max(input_len + output_len) */
  int64_t sum_input;
  int64_t sum_output;
} arrow_synth_result_t;

/* Generate n_traces traces.  Request k of trace i is written to
 * arrival/input_len/output_len[specs[i].out_offset + k] for k < capacity. */
int arrow_synth_run(const arrow_synth_t* specs, int32_t n_traces, double* arrival, int32_t* input_len,
                    int32_t* output_len, arrow_synth_result_t* results, void* stream);

/* sizeof(arrow_synth_t), sizeof(arrow_synth_result_t) and every field
 * offset in declaration order.  Returns the number of values. */
int arrow_synth_layout(int64_t* out, int cap);

/* ---- trace statistics (§8(f) rank 4) ------------------------------------
 * Replaces the per-request scan of
 *     pdsim.traces.trace_stats(trace, bucket_s)            traces.py:202-250
 * with one streaming pass over the SoA trace (16 B per request): per-bucket
 * request / input / output totals (bucket = int(arrival // bucket_s) with
 * CPython's float floor division), first/last arrival with Python min/max
 * tie semantics, exact integer moments for the Pearson r, and exact
 * histograms of the lengths for np.percentile's order statistics.  The host
 * turns these into TraceStats with the reference's own formulas. */

#define ARROW_STATS_HIST_BINS 16384   /* lengths 1..16384 counted exactly in the scan */

typedef struct arrow_stats_partial {  /* one per block; merged on the host */
  double min_arrival;         /* NaN: block saw nothing */
  double max_arrival;
  int64_t count;              /* requests counted into buckets */
  int64_t sum_x, sum_y;       /* x = input_len, y = output_len (bucketed requests) */
  uint64_t sxx_lo, sxx_hi;    /* 128-bit sums of x*x, y*y, x*y */
  uint64_t syy_lo, syy_hi;
  uint64_t sxy_lo, sxy_hi;
  int64_t out_of_window;      /* requests whose bucket fell outside [bucket_lo, bucket_lo + n_buckets) */
} arrow_stats_partial_t;

typedef struct arrow_stats_args {
  const double* arrival;
  const int32_t* input_len;
  const int32_t* output_len;
  int64_t n;
  double bucket_s;            /* > 0 */
  int64_t bucket_lo;          /* int(first // bucket_s), |bucket_lo| < 2^53 */
  int64_t n_buckets;          /* hi - lo + 1 */
  int64_t* bucket_requests;   /* [n_buckets] each, zeroed by arrow_stats_run */
  int64_t* bucket_input;
  int64_t* bucket_output;
  uint32_t* hist_x;           /* [ARROW_STATS_HIST_BINS], bin v - 1; zeroed by arrow_stats_run */
  uint32_t* hist_y;
  arrow_stats_partial_t* partials;
  int32_t n_partials;         /* grid size; arrow_stats_grid() gives the preferred value */
  int32_t reserved;
} arrow_stats_args_t;

/* Preferred number of partials (blocks) for n requests on the current device. */
int arrow_stats_grid(int64_t n, int32_t* n_partials);

int arrow_stats_run(const arrow_stats_args_t* args, void* stream);

/* Radix step for order statistics beyond the exact bins: counts values v of
 * [values, values + n) with lo <= v < hi into bins[(v - lo) >> shift]
 * (bins zeroed here, n_bins = ((hi - lo - 1) >> shift) + 1). */
int arrow_stats_hist(const int32_t* values, int64_t n, int64_t lo, int64_t hi, int32_t shift, uint32_t* bins,
                     int64_t n_bins, void* stream);

int arrow_stats_layout(int64_t* out, int cap);

#ifdef __cplusplus
}
#endif

#endif /* ARROW_TRACES_H */
