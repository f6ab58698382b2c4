// traces.cu — device workload generator + C-ABI (include/arrow_traces.h).
//
// One thread = one trace: the reference's generator is a single sequential
// PCG64 stream whose consumption per candidate arrival depends on the
// thinning outcome and on the ziggurats' rare paths (traces.py:159-175), so
// a trace cannot be split without changing its numbers; batches of
// (params, seed) pairs are the parallel axis.  The ziggurat and exp tables
// (14 KB) are staged in shared memory once per block, which keeps the
// data-dependent table lookups of 32 different streams per warp off the
// serialising constant cache.  Requests are written straight into the
// caller's per-trace slices of the SoA trace arrays the evaluator reads.
#include <cuda_runtime.h>
#include <stddef.h>

#include "arrow_traces.h"
#define NPGEN_STORAGE static __device__ const
#include "npgen.cuh"

namespace {

#ifndef ARROW_GEN_THREADS
#define ARROW_GEN_THREADS 128
#endif
constexpr int kGenThreads = ARROW_GEN_THREADS;

__global__ void __launch_bounds__(kGenThreads) arrow_synth_kernel(const arrow_synth_t* __restrict__ specs, int n_traces,
                                                                  double* __restrict__ arrival,
                                                                  int32_t* __restrict__ input_len,
                                                                  int32_t* __restrict__ output_len,
                                                                  arrow_synth_result_t* __restrict__ results) {
  __shared__ uint64_t tab[7][256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    tab[0][i] = npgen::KE_DOUBLE_BITS[i];
    tab[1][i] = npgen::WE_DOUBLE_BITS[i];
    tab[2][i] = npgen::FE_DOUBLE_BITS[i];
    tab[3][i] = npgen::KI_DOUBLE_BITS[i];
    tab[4][i] = npgen::WI_DOUBLE_BITS[i];
    tab[5][i] = npgen::FI_DOUBLE_BITS[i];
    tab[6][i] = npgen::EXP_TAB[i];
  }
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_traces) return;
  const npgen::Tables T{tab[0], tab[1], tab[2], tab[3], tab[4], tab[5], tab[6]};
  const arrow_synth_t& P = specs[i];
  const int64_t off = P.out_offset;
  const int64_t cap = P.capacity;
  double first = __longlong_as_double(0x7ff8000000000000ll), last = first;
  int64_t max_kv = 0, sum_in = 0, sum_out = 0;
  int status = ARROW_SYNTH_OK;
  const int64_t n = npgen::gen_synthetic(
      P, T,
      [&](int64_t k, double t, int64_t in, int64_t out) {
        if (k == 0) first = t;
        last = t;
        max_kv = max(max_kv, in + out);
        sum_in += in;
        sum_out += out;
        if (k < cap) {
          arrival[off + k] = t;
          input_len[off + k] = (int32_t)in;
          output_len[off + k] = (int32_t)out;
        }
      },
      &status);
  arrow_synth_result_t r;
  r.count = n;
  r.status = (status == ARROW_SYNTH_OK && n > cap) ? ARROW_SYNTH_CAPACITY : status;
  r.reserved = 0;
  r.first_arrival = first;
  r.last_arrival = last;
  r.max_kv = max_kv;
  r.sum_input = sum_in;
  r.sum_output = sum_out;
  results[i] = r;
}

}  // namespace

extern "C" {

int arrow_synth_run(const arrow_synth_t* specs, int32_t n_traces, double* arrival, int32_t* input_len,
                    int32_t* output_len, arrow_synth_result_t* results, void* stream) {
  if (n_traces <= 0) return 0;
  const int blocks = (n_traces + kGenThreads - 1) / kGenThreads;
  arrow_synth_kernel<<<blocks, kGenThreads, 0, (cudaStream_t)stream>>>(specs, n_traces, arrival, input_len,
                                                                        output_len, results);
  return (int)cudaGetLastError();
}

int arrow_synth_layout(int64_t* out, int cap) {
  int64_t v[64];
  int n = 0;
#define SZ(T) v[n++] = (int64_t)sizeof(T)
#define OFF(T, f) v[n++] = (int64_t)offsetof(T, f)
  SZ(arrow_synth_t);
  SZ(arrow_synth_result_t);
  OFF(arrow_synth_t, duration_s);
  OFF(arrow_synth_t, base_rate);
  OFF(arrow_synth_t, rate_max);
  OFF(arrow_synth_t, gap_scale);
  OFF(arrow_synth_t, input_log_mean);
  OFF(arrow_synth_t, input_log_sigma);
  OFF(arrow_synth_t, output_log_mean);
  OFF(arrow_synth_t, output_log_sigma);
  OFF(arrow_synth_t, max_input);
  OFF(arrow_synth_t, max_output);
  OFF(arrow_synth_t, n_bursts);
  OFF(arrow_synth_t, n_seed_words);
  OFF(arrow_synth_t, seed_words);
  OFF(arrow_synth_t, burst_start);
  OFF(arrow_synth_t, burst_duration);
  OFF(arrow_synth_t, burst_multiplier);
  OFF(arrow_synth_t, out_offset);
  OFF(arrow_synth_t, capacity);
  OFF(arrow_synth_result_t, count);
  OFF(arrow_synth_result_t, status);
  OFF(arrow_synth_result_t, reserved);
  OFF(arrow_synth_result_t, first_arrival);
  OFF(arrow_synth_result_t, last_arrival);
  OFF(arrow_synth_result_t, max_kv);
  OFF(arrow_synth_result_t, sum_input);
  OFF(arrow_synth_result_t, sum_output);
#undef SZ
#undef OFF
  for (int i = 0; i < n && i < cap; i++) out[i] = v[i];
  return n;
}

}  // extern "C"
