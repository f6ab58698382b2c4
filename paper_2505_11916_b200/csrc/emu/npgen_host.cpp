// npgen_host.cpp — TEST-ONLY host build of the device generator source
// (csrc/npgen.cuh).  The CPU tests load it to check, without a GPU, that the
// very code the CUDA kernel runs reproduces numpy's PCG64 / SeedSequence /
// ziggurat streams, glibc's exp / log1p and the reference's gen_synthetic
// bit for bit.  Never loaded by the product path.
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "arrow_traces.h"
#include "../npgen.cuh"

namespace {

npgen::Tables host_tables() {
  return npgen::Tables{npgen::KE_DOUBLE_BITS, npgen::WE_DOUBLE_BITS, npgen::FE_DOUBLE_BITS, npgen::KI_DOUBLE_BITS,
                       npgen::WI_DOUBLE_BITS, npgen::FI_DOUBLE_BITS, npgen::EXP_TAB};
}

npgen::Pcg64 from_words(const uint64_t* s) {
  npgen::Pcg64 g;
  g.state = npgen::U128{s[0], s[1]};
  g.inc = npgen::U128{s[2], s[3]};
  return g;
}

void to_words(const npgen::Pcg64& g, uint64_t* s) {
  s[0] = g.state.hi;
  s[1] = g.state.lo;
  s[2] = g.inc.hi;
  s[3] = g.inc.lo;
}

// xorshift64* stream for the libm sweeps
uint64_t mix64(uint64_t& x) {
  x ^= x >> 12;
  x ^= x << 25;
  x ^= x >> 27;
  return x * 0x2545F4914F6CDD1Dull;
}

}  // namespace

extern "C" {

double npgen_log1p(double x) { return npgen::glibc_log1p(x); }
double npgen_exp(double x) { return npgen::glibc_exp(x, npgen::EXP_TAB); }

// PCG64 state (state.hi, state.lo, inc.hi, inc.lo) of default_rng(seed).
void npgen_seed_state(const uint32_t* words, int n_words, uint64_t* out4) {
  uint64_t s[4];
  npgen::seed_sequence_u64x4(words, n_words, s);
  npgen::Pcg64 g;
  g.seed(s);
  to_words(g, out4);
}

// kind 0: raw uint64, 1: random(), 2: standard_exponential, 3: standard_normal.
// state4 is advanced in place.
void npgen_draw(uint64_t* state4, int kind, int64_t n, void* out) {
  npgen::Pcg64 g = from_words(state4);
  const npgen::Tables T = host_tables();
  for (int64_t i = 0; i < n; i++) {
    switch (kind) {
      case 0: ((uint64_t*)out)[i] = g.next64(); break;
      case 1: ((double*)out)[i] = g.next_double(); break;
      case 2: ((double*)out)[i] = npgen::standard_exponential(g, T); break;
      default: ((double*)out)[i] = npgen::standard_normal(g, T); break;
    }
  }
  to_words(g, state4);
}

// Compare against the process's libm on n inputs: kind 0 log1p(-u) for
// u in [0,1) (the samplers' domain), 1 log1p on random bit patterns in
// (-1, 2^60), 2 exp on [-745, 710], 3 exp on random finite bit patterns,
// 4 exp on [-8, 12] (the lengths' and rejection tests' domain).
// Returns mismatches; the first is stored in *bad_x.
int64_t npgen_check_libm(int kind, int64_t n, uint64_t seed, double* bad_x) {
  uint64_t st = seed | 1;
  int64_t bad = 0;
  for (int64_t i = 0; i < n; i++) {
    const uint64_t r = mix64(st);
    double x, a, b;
    if (kind == 0) {
      x = -((double)(r >> 11) * (1.0 / 9007199254740992.0));
      a = npgen::glibc_log1p(x);
      b = log1p(x);
    } else if (kind == 1) {
      x = npgen::from_bits(r & 0x7fffffffffffffffull);
      if (r >> 63) x = -npgen::from_bits(r & 0x3fefffffffffffffull);  // (-1, 0)
      if (!(x < 0x1p60)) x = 1.5;
      a = npgen::glibc_log1p(x);
      b = log1p(x);
    } else if (kind == 2) {
      x = -745.0 + 1455.0 * ((double)(r >> 11) * (1.0 / 9007199254740992.0));
      a = npgen::glibc_exp(x, npgen::EXP_TAB);
      b = exp(x);
    } else if (kind == 3) {
      x = npgen::from_bits(r);
      if (isnan(x)) x = 0.5;
      a = npgen::glibc_exp(x, npgen::EXP_TAB);
      b = exp(x);
    } else {
      x = -8.0 + 20.0 * ((double)(r >> 11) * (1.0 / 9007199254740992.0));
      a = npgen::glibc_exp(x, npgen::EXP_TAB);
      b = exp(x);
    }
    if (npgen::bits_of(a) != npgen::bits_of(b) && !(isnan(a) && isnan(b))) {
      if (bad == 0 && bad_x) *bad_x = x;
      bad++;
    }
  }
  return bad;
}

// Same contract as arrow_synth_run, on host memory.
int npgen_synth_run(const arrow_synth_t* specs, int32_t n_traces, double* arrival, int32_t* input_len,
                    int32_t* output_len, arrow_synth_result_t* results) {
  const npgen::Tables T = host_tables();
  for (int i = 0; i < n_traces; i++) {
    const arrow_synth_t& P = specs[i];
    double first = NAN, last = NAN;
    int64_t max_kv = 0, sum_in = 0, sum_out = 0;
    int status = 0;
    const int64_t n = npgen::gen_synthetic(
        P, T,
        [&](int64_t k, double t, int64_t in, int64_t out) {
          if (k == 0) first = t;
          last = t;
          if (in + out > max_kv) max_kv = in + out;
          sum_in += in;
          sum_out += out;
          if (k < P.capacity) {
            arrival[P.out_offset + k] = t;
            input_len[P.out_offset + k] = (int32_t)in;
            output_len[P.out_offset + k] = (int32_t)out;
          }
        },
        &status);
    arrow_synth_result_t& r = results[i];
    r.count = n;
    r.status = (status == ARROW_SYNTH_OK && n > P.capacity) ? ARROW_SYNTH_CAPACITY : status;
    r.reserved = 0;
    r.first_arrival = first;
    r.last_arrival = last;
    r.max_kv = max_kv;
    r.sum_input = sum_in;
    r.sum_output = sum_out;
  }
  return 0;
}

}  // extern "C"
