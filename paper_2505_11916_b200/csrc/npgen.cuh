// npgen.cuh — numpy's Generator(PCG64) streams and the reference's synthetic
// workload generator, bit for bit, for the device (and, for tests, the host).
//
// The reference draws every synthetic trace with
//     rng = np.random.default_rng(seed)                        traces.py:161
//     t += rng.exponential(1 / rate_max)                       traces.py:166
//     if rng.random() * rate_max > _rate_at(t): continue       traces.py:169-170
//     x = math.exp(rng.normal(mu, sigma))                      traces.py:154-156
//     int(min(max(round(x), 1), max_len))
// so reproducing a trace means reproducing, in order:
//   * SeedSequence(seed) -> 4 x uint64 -> PCG64 state/increment
//     (numpy/random/bit_generator.pyx, numpy/random/_pcg64.pyx),
//   * PCG64 XSL-RR 128/64 (state advanced before output),
//   * random_standard_uniform  = (next64 >> 11) * 2^-53,
//   * random_standard_exponential / random_standard_normal: 256-level
//     ziggurats with numpy's tables (npgen_tables.h) and their rare paths,
//     which call the C library's log1p and exp,
//   * CPython's math.exp and round() (half-even).
// log1p and exp are therefore restated here exactly as the x86-64 glibc 2.39
// FMA variants compute them (the variant the image's libm selects on
// FMA-capable CPUs): same polynomial, same table, same fused operations, so
// the results are identical, not merely within an ulp.  Everything else is
// plain IEEE double without contraction (-fmad=false / -ffp-contract=off);
// the fused operations below are explicit fma() calls.
#pragma once

#include <math.h>
#include <stdint.h>
#include <string.h>

#include "warp.cuh"  // AS_HD

#ifndef NPGEN_STORAGE
#define NPGEN_STORAGE static const
#endif
#include "npgen_tables.h"

namespace npgen {

AS_HD uint64_t bits_of(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
}

AS_HD double from_bits(uint64_t u) {
  double x;
  memcpy(&x, &u, 8);
  return x;
}

AS_HD double with_hi(double x, uint32_t hi) {
  return from_bits((bits_of(x) & 0xffffffffull) | ((uint64_t)hi << 32));
}

// Tables, resident wherever the caller put them (shared memory on the device).
struct Tables {
  const uint64_t* ke;
  const uint64_t* we;
  const uint64_t* fe;
  const uint64_t* ki;
  const uint64_t* wi;
  const uint64_t* fi;
  const uint64_t* exp_tab;
};

// ------------------------------------------------------------ glibc libm --

// log1p, sysdeps/ieee754/dbl-64/s_log1p.c as built for x86-64 with FMA
// (Lp1..Lp7 evaluated Estrin-style; fused where the FMA build fuses).
AS_HD double glibc_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01;
  const double Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01;
  const double Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01;
  const double Lp7 = 1.479819860511658591e-01;
  const int32_t hx = (int32_t)(bits_of(x) >> 32);
  const int32_t ax = hx & 0x7fffffff;
  int k = 1;
  int32_t hu = 0;
  double f = 0.0, c = 0.0, u;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) {
      if (x == -1.0) return -INFINITY;
      return NAN;
    }
    if (ax < 0x3e200000) {
      if (ax < 0x3c900000) return x;
      const double xx = x * x;
      return fma(-xx, 0.5, x);
    }
    if (hx > 0 || hx <= (int32_t)0xbfd2bec3) {
      k = 0;
      f = x;
      hu = 1;
    }
  } else if (hx >= 0x7ff00000) {
    return x + x;
  }
  if (k != 0) {
    if (hx < 0x43400000) {
      u = 1.0 + x;
      hu = (int32_t)(bits_of(u) >> 32);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);
      c = c / u;
    } else {
      u = x;
      hu = hx;
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = with_hi(u, (uint32_t)(hu | 0x3ff00000));
    } else {
      k += 1;
      u = with_hi(u, (uint32_t)(hu | 0x3fe00000));
      hu = (0x00100000 - hu) >> 2;
    }
    f = u - 1.0;
  }
  const double hfsq = (f * 0.5) * f;
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      const double kd = (double)k;
      return fma(kd, ln2_hi, fma(kd, ln2_lo, c));
    }
    const double R = fma(-f, 0.66666666666666666, 1.0) * hfsq;
    if (k == 0) return f - R;
    const double kd = (double)k;
    return fma(kd, ln2_hi, -((R - fma(kd, ln2_lo, c)) - f));
  }
  const double s = f / (2.0 + f);
  const double z = s * s;
  const double R2 = fma(z, Lp3, Lp2);
  const double R3 = fma(z, Lp5, Lp4);
  const double R4 = fma(z, Lp7, Lp6);
  const double z2 = z * z;
  const double z4 = z2 * z2;
  const double z6 = z2 * z4;
  double R = z2 * R2;
  R = fma(z, Lp1, R);
  R = fma(z4, R3, R);
  R = fma(z6, R4, R);
  const double w = (R + hfsq) * s;
  if (k == 0) return f - (hfsq - w);
  const double kd = (double)k;
  const double t = (hfsq - (fma(kd, ln2_lo, c) + w)) - f;
  return fma(kd, ln2_hi, -t);
}

// exp, sysdeps/ieee754/dbl-64/e_exp.c (optimized-routines, 128-entry
// table) as built for x86-64 with FMA.
AS_HD double glibc_exp(double x, const uint64_t* T) {
  const double InvLn2N = 0x1.71547652b82fep7;
  const double Shift = 0x1.8p52;
  const double NegLn2hiN = -0x1.62e42fefa0000p-8;
  const double NegLn2loN = -0x1.cf79abc9e3b3ap-47;
  const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3;
  const double C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;
  const uint64_t ux = bits_of(x);
  uint32_t abstop = (uint32_t)(ux >> 52) & 0x7ff;
  if (abstop - 0x3c9u >= 0x3fu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) return x + 1.0;
    if (abstop >= 0x409u) {
      if (ux == 0xfff0000000000000ull) return 0.0;
      if (abstop >= 0x7ffu) return x + 1.0;
      return (ux >> 63) ? 0.0 : INFINITY;
    }
    abstop = 0;
  }
  double kd = fma(x, InvLn2N, Shift);
  const uint64_t ki = bits_of(kd);
  kd = kd - Shift;
  double r = fma(kd, NegLn2hiN, x);
  r = fma(kd, NegLn2loN, r);
  const uint64_t idx = 2 * (ki & 127);
  const uint64_t top = ki << 45;
  const double tail = from_bits(T[idx]);
  uint64_t sbits = T[idx + 1] + top;
  const double p23 = fma(r, C3, C2);
  const double tr = r + tail;
  const double r2 = r * r;
  const double p45 = fma(r, C5, C4);
  double tmp = fma(p23, r2, tr);
  const double r4 = r2 * r2;
  tmp = fma(r4, p45, tmp);
  if (abstop == 0) {
    // specialcase(): scale out of the normal range
    if ((ki & 0x80000000ull) == 0) {
      sbits -= 1009ull << 52;
      const double scale = from_bits(sbits);
      return fma(scale, tmp, scale) * 0x1p1009;
    }
    sbits += 1022ull << 52;
    const double scale = from_bits(sbits);
    const double st = tmp * scale;
    double y = scale + st;
    if (1.0 > y) {
      const double hi = y + 1.0;
      const double lo = (scale - y) + st;
      double z = ((1.0 - hi) + y) + lo;
      z = z + hi;
      y = z - 1.0;
      if (y == 0.0) return 0.0;
    }
    return y * 0x1p-1022;
  }
  const double scale = from_bits(sbits);
  return fma(scale, tmp, scale);
}

// ------------------------------------------------------- SeedSequence ---

// numpy/random/bit_generator.pyx: pool of 4 uint32 words, hashmix / mix.
struct SeedHash {
  uint32_t c;
  AS_HD uint32_t hashmix(uint32_t v) {
    v ^= c;
    c *= 0x931e8875u;  // MULT_A
    v *= c;
    v ^= v >> 16;
    return v;
  }
};

AS_HD uint32_t seed_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;  // MIX_MULT_L, MIX_MULT_R
  r ^= r >> 16;
  return r;
}

// SeedSequence(entropy).generate_state(4, uint64); entropy = the seed's
// little-endian uint32 words (_int_to_uint32_array), no spawn key.
AS_HD void seed_sequence_u64x4(const uint32_t* ent, int n_ent, uint64_t out[4]) {
  uint32_t pool[4];
  SeedHash h{0x43b0d7e5u};  // INIT_A
  for (int i = 0; i < 4; i++) pool[i] = h.hashmix(i < n_ent ? ent[i] : 0u);
  for (int s = 0; s < 4; s++)
    for (int d = 0; d < 4; d++)
      if (s != d) pool[d] = seed_mix(pool[d], h.hashmix(pool[s]));
  for (int s = 4; s < n_ent; s++)
    for (int d = 0; d < 4; d++) pool[d] = seed_mix(pool[d], h.hashmix(ent[s]));
  uint32_t hc = 0x8b51f9ddu;  // INIT_B
  uint32_t w[8];
  for (int i = 0; i < 8; i++) {
    uint32_t v = pool[i & 3];
    v ^= hc;
    hc *= 0x58f38dedu;  // MULT_B
    v *= hc;
    v ^= v >> 16;
    w[i] = v;
  }
  for (int j = 0; j < 4; j++) out[j] = (uint64_t)w[2 * j] | ((uint64_t)w[2 * j + 1] << 32);
}

// ------------------------------------------------------------- PCG64 ----

struct U128 {
  uint64_t hi, lo;
};

AS_HD U128 mul128(U128 a, U128 b) {
#ifdef __CUDA_ARCH__
  const uint64_t hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return U128{hi, a.lo * b.lo};
#else
  const unsigned __int128 p = (unsigned __int128)a.lo * b.lo;
  return U128{(uint64_t)(p >> 64) + a.lo * b.hi + a.hi * b.lo, (uint64_t)p};
#endif
}

AS_HD U128 add128(U128 a, U128 b) {
  const uint64_t lo = a.lo + b.lo;
  return U128{a.hi + b.hi + (lo < a.lo ? 1u : 0u), lo};
}

// numpy/random/src/pcg64: PCG_DEFAULT_MULTIPLIER_128, XSL-RR output of the
// advanced state.
struct Pcg64 {
  U128 state, inc;

  AS_HD void step() {
    state = add128(mul128(state, U128{0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull}), inc);
  }
  AS_HD uint64_t next64() {
    step();
    const uint64_t x = state.hi ^ state.lo;
    const unsigned rot = (unsigned)(state.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  AS_HD double next_double() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }

  // pcg64_set_seed: seed = (s[0] << 64) | s[1], inc = (s[2] << 64) | s[3]
  AS_HD void seed(const uint64_t s[4]) {
    state = U128{0, 0};
    inc = U128{(s[2] << 1) | (s[3] >> 63), (s[3] << 1) | 1u};
    step();
    state = add128(state, U128{s[0], s[1]});
    step();
  }
};

// ------------------------------------------------ Generator samplers ----

static constexpr double ZIG_EXP_R = 0x1.ec9d9297ebb83p+2;      // 7.69711747013104972
static constexpr double ZIG_NOR_R = 0x1.d3bb48209ad33p+1;      // 3.6541528853610088
static constexpr double ZIG_NOR_INV_R = 0x1.183aa6c20e8c1p-2;  // 0.27366123732975828

// random_standard_exponential (distributions.c)
AS_HD double standard_exponential(Pcg64& g, const Tables& T) {
  for (;;) {
    uint64_t ri = g.next64();
    ri >>= 3;
    const int idx = (int)(ri & 0xff);
    ri >>= 8;
    const double x = (double)ri * from_bits(T.we[idx]);
    if (ri < T.ke[idx]) return x;
    if (idx == 0) return ZIG_EXP_R - glibc_log1p(-g.next_double());
    const double fe0 = from_bits(T.fe[idx - 1]), fe1 = from_bits(T.fe[idx]);
    const double u = g.next_double();
    if ((fe0 - fe1) * u + fe1 < glibc_exp(-x, T.exp_tab)) return x;
  }
}

// random_standard_normal (distributions.c)
AS_HD double standard_normal(Pcg64& g, const Tables& T) {
  for (;;) {
    uint64_t r = g.next64();
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * from_bits(T.wi[idx]);
    if (sign) x = -x;
    if (rabs < T.ki[idx]) return x;
    if (idx == 0) {
      for (;;) {
        const double xx = -ZIG_NOR_INV_R * glibc_log1p(-g.next_double());
        const double yy = -glibc_log1p(-g.next_double());
        if (yy + yy > xx * xx) return ((rabs >> 8) & 1) ? -(ZIG_NOR_R + xx) : ZIG_NOR_R + xx;
      }
    }
    const double fi0 = from_bits(T.fi[idx - 1]), fi1 = from_bits(T.fi[idx]);
    const double u = g.next_double();
    if ((fi0 - fi1) * u + fi1 < glibc_exp(-0.5 * x * x, T.exp_tab)) return x;
  }
}

// ---------------------------------------------- the reference's loop ----

// CPython round() on a float (half-even) then int(min(max(v, 1), cap))
// (traces.py:154-156).  x = inf (math.exp overflowed: OverflowError in the
// reference) is the caller's to check.
AS_HD int64_t clamp_length(double x, int64_t cap) {
  const double v = rint(x);
  if (v < 1.0) return 1 < cap ? 1 : cap;
  if (v >= (double)cap) return cap;
  return (int64_t)v;
}

}  // namespace npgen

// ------------------------------------------------------------------------
// gen_synthetic (traces.py:159-175) for one arrow_synth_t.  emit(k, t, in,
// out) receives every accepted request in order; returns the request count
// and sets *status (arrow_synth_status).
#ifdef ARROW_TRACES_H
namespace npgen {

AS_HD double rate_at(const arrow_synth_t& P, double t) {  // traces.py:146-151
  double rate = P.base_rate;
  for (int b = 0; b < P.n_bursts; b++)
    if (P.burst_start[b] <= t && t < P.burst_start[b] + P.burst_duration[b]) rate *= P.burst_multiplier[b];
  return rate;
}

template <class Emit>
AS_HD int64_t gen_synthetic(const arrow_synth_t& P, const Tables& T, Emit&& emit, int* status) {
  uint64_t s[4];
  seed_sequence_u64x4(P.seed_words, P.n_seed_words, s);
  Pcg64 g;
  g.seed(s);
  double t = 0.0;
  int64_t n = 0;
  *status = ARROW_SYNTH_OK;
  for (;;) {
    t += P.gap_scale * standard_exponential(g, T);
    if (t >= P.duration_s) break;
    if (g.next_double() * P.rate_max > rate_at(P, t)) continue;
    const double xi = glibc_exp(P.input_log_mean + P.input_log_sigma * standard_normal(g, T), T.exp_tab);
    if (xi == INFINITY) {
      *status = ARROW_SYNTH_OVERFLOW;
      break;
    }
    const double xo = glibc_exp(P.output_log_mean + P.output_log_sigma * standard_normal(g, T), T.exp_tab);
    if (xo == INFINITY) {
      *status = ARROW_SYNTH_OVERFLOW;
      break;
    }
    emit(n, t, clamp_length(xi, P.max_input), clamp_length(xo, P.max_output));
    n++;
  }
  return n;
}

}  // namespace npgen
#endif
