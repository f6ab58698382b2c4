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

#ifdef __cplusplus
}
#endif

#endif /* ARROW_TRACES_H */
