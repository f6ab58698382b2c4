// stats.cu — trace statistics scan + C-ABI (include/arrow_traces.h).
//
// trace_stats (traces.py:202-250) is a pure scan: every request is read once
// (arrival f64, input i32, output i32 = 16 B) and folded into
//   * per-bucket totals, bucket = int(arrival // bucket_s) (CPython float
//     floor division, reproduced exactly).  Each warp owns one contiguous
//     range of the trace and keeps per-lane running totals for its current
//     bucket; only when the bucket changes are they warp-reduced and added
//     to HBM with three atomics.  A sorted trace therefore costs a handful of
//     register adds per request and one flush per bucket boundary per warp;
//     slices straddling buckets (or unsorted traces) fall back to
//     __match_any_sync-grouped atomics;
//   * exact histograms of the lengths 1..16384 in shared memory (flushed
//     once per block) -> np.percentile's order statistics;
//   * exact 64/128-bit integer moments (x^2, y^2, xy) -> the Pearson r;
//   * min / max arrival.  (Python's min/max return the first of equal
//     values, which differs only in the sign of a zero; no TraceStats field
//     can observe it: the duration of an all-zero trace is z - z = +0.0.)
// One persistent block per SM (the 128 KB histogram fills its shared
// memory), 16 warps streaming 256-request chunks: every lane issues 24
// independent coalesced loads before using any.
#include <cuda_runtime.h>
#include <math.h>
#include <stddef.h>
#include <stdint.h>

#include "arrow_traces.h"

namespace {

#ifndef ARROW_STATS_THREADS
#define ARROW_STATS_THREADS 512
#endif
constexpr int kStatsThreads = ARROW_STATS_THREADS;
#ifndef ARROW_STATS_PER
#define ARROW_STATS_PER 4
#endif
constexpr int kPer = ARROW_STATS_PER;   // requests per lane per chunk (one ring stage)
constexpr int kChunk = 32 * kPer;
constexpr int kWarps = kStatsThreads / 32;
constexpr int kBins = ARROW_STATS_HIST_BINS;
constexpr uint32_t FULL = 0xffffffffu;

// CPython float_floor_div (Objects/floatobject.c, _float_div_mod), general path.
__device__ __noinline__ double py_floordiv(double vx, double wx) {
  double mod = fmod(vx, wx);
  double div = (vx - mod) / wx;
  if (mod != 0.0) {
    if ((wx < 0) != (mod < 0)) div -= 1.0;
  }
  double fd;
  if (div != 0.0) {
    fd = floor(div);
    if (div - fd > 0.5) fd += 1.0;
  } else {
    fd = copysign(0.0, vx / wx);
  }
  return fd;
}

// Fast path of the same: for vx >= 0, wx > 0 and a quotient below 2^50,
// CPython returns trunc() of the EXACT quotient (fmod is exact, vx - mod =
// m*wx rounds by at most 2^-53 relative, the division adds 2^-53, and the
// final snap to the nearest integer absorbs both while m < 2^51).  That
// integer is found without fmod's bit-serial loop: floor(vx * (1/wx)) is
// within one of it and exact-sign FMA residuals vx - m*wx correct it.
// ok = false sends the caller to py_floordiv.
__device__ __forceinline__ double floordiv_fast(double vx, double wx, double inv, bool& ok) {
  const double q = vx * inv;
  ok = vx >= 0.0 && q < 0x1p50;
  double m = floor(q);
  if (fma(-m, wx, vx) < 0.0)
    m -= 1.0;
  else if (fma(-(m + 1.0), wx, vx) >= 0.0)
    m += 1.0;
  return m;
}

struct U128 {
  uint64_t lo, hi;
  __device__ __forceinline__ void add(uint64_t v) {
    lo += v;
    hi += (lo < v) ? 1u : 0u;
  }
  __device__ __forceinline__ void add(U128 o) {
    lo += o.lo;
    hi += o.hi + ((lo < o.lo) ? 1u : 0u);
  }
};

struct Acc {
  double tmin, tmax;
  int64_t count, sx, sy, oow;
  U128 sxx, syy, sxy;
  uint64_t pxx, pyy, pxy;  // pending 64-bit moments of up to 32/kPer chunks
  int pn;

  __device__ void init() {
    tmin = INFINITY;
    tmax = -INFINITY;
    count = sx = sy = oow = 0;
    sxx = syy = sxy = U128{0, 0};
    pxx = pyy = pxy = 0;
    pn = 0;
  }
  __device__ void flush_pending() {
    sxx.add(pxx);
    syy.add(pyy);
    sxy.add(pxy);
    pxx = pyy = pxy = 0;
    pn = 0;
  }
  __device__ void merge(const Acc& o) {
    tmin = fmin(tmin, o.tmin);
    tmax = fmax(tmax, o.tmax);
    count += o.count;
    sx += o.sx;
    sy += o.sy;
    oow += o.oow;
    sxx.add(o.sxx);
    syy.add(o.syy);
    sxy.add(o.sxy);
  }
};

template <class T>
__device__ __forceinline__ T shfl_down(T v, int d) {
  return __shfl_down_sync(FULL, v, d);
}

__device__ void warp_merge(Acc& a) {
  for (int d = 16; d > 0; d >>= 1) {
    Acc o;
    o.tmin = shfl_down(a.tmin, d);
    o.tmax = shfl_down(a.tmax, d);
    o.count = shfl_down(a.count, d);
    o.sx = shfl_down(a.sx, d);
    o.sy = shfl_down(a.sy, d);
    o.oow = shfl_down(a.oow, d);
    o.sxx = U128{shfl_down(a.sxx.lo, d), shfl_down(a.sxx.hi, d)};
    o.syy = U128{shfl_down(a.syy.lo, d), shfl_down(a.syy.hi, d)};
    o.sxy = U128{shfl_down(a.sxy.lo, d), shfl_down(a.sxy.hi, d)};
    a.merge(o);
  }
}

// Each histogram is kBins + 2 words indexed by the length itself: word v for
// v in 1..kBins, word 0 (v == 0) and word kBins + 1 (v > kBins, or v < 0 as
// unsigned) are spares the copy-out skips.  One unsigned min, one address
// and one unconditional red.shared per update (no branch, no generic-to-
// shared conversion).
constexpr int kHistSpan = kBins + 2;
constexpr int kHistWords = (2 * kHistSpan + 31) / 32 * 32;  // keeps the ring 128 B aligned
__device__ __forceinline__ void hist_inc(uint32_t hist_sa, int32_t v) {
  const uint32_t idx = min((uint32_t)v, (uint32_t)(kBins + 1));
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(hist_sa + 4u * idx) : "memory");
}

__device__ __forceinline__ uint64_t warp_sum(uint64_t v) {
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
  return v;
}

// Per-lane running totals of the warp's current bucket.
struct Run {
  double f, f1;      // bucket (as the floor-division double) and f + 1, warp-uniform; NaN = none
  uint32_t c;        // requests
  uint64_t x, y;     // input / output tokens

  __device__ void flush(const arrow_stats_args_t& A, Acc& acc, double lo_d, int lane) {
    const uint64_t sc = warp_sum(c), sx = warp_sum(x), sy = warp_sum(y);
    if (lane == 0 && sc) {
      const int64_t b = (int64_t)(f - lo_d);
      atomicAdd((unsigned long long*)&A.bucket_requests[b], (unsigned long long)sc);
      atomicAdd((unsigned long long*)&A.bucket_input[b], (unsigned long long)sx);
      atomicAdd((unsigned long long*)&A.bucket_output[b], (unsigned long long)sy);
      acc.count += (int64_t)sc;
      acc.sx += (int64_t)sx;
      acc.sy += (int64_t)sy;
    }
    c = 0;
    x = y = 0;
  }
};

// Lanes holding the same bucket add their totals with one atomic per bucket.
__device__ __forceinline__ void bucket_add(const arrow_stats_args_t& A, Acc& acc, int64_t b, int32_t x, int32_t y,
                                           int lane) {
  const unsigned long long key = (unsigned long long)b;
  const uint32_t peers = __match_any_sync(FULL, key);
  if (b < 0) return;
  const uint32_t ux = (uint32_t)x, uy = (uint32_t)y;
  const uint64_t sx = (uint64_t)__reduce_add_sync(peers, ux & 0xffffu) +
                      ((uint64_t)__reduce_add_sync(peers, ux >> 16) << 16);
  const uint64_t sy = (uint64_t)__reduce_add_sync(peers, uy & 0xffffu) +
                      ((uint64_t)__reduce_add_sync(peers, uy >> 16) << 16);
  if (lane == __ffs(peers) - 1) {
    atomicAdd((unsigned long long*)&A.bucket_requests[b], (unsigned long long)__popc(peers));
    atomicAdd((unsigned long long*)&A.bucket_input[b], (unsigned long long)sx);
    atomicAdd((unsigned long long*)&A.bucket_output[b], (unsigned long long)sy);
    acc.count += __popc(peers);
    acc.sx += (int64_t)sx;
    acc.sy += (int64_t)sy;
  }
}

// A warp's chunk of 32*kPer requests held in registers.
struct Chunk {
  double t[kPer];
  int32_t x[kPer], y[kPer];
};

__device__ __forceinline__ void load_chunk(const arrow_stats_args_t& A, Chunk& c, int64_t base, int64_t end,
                                           int lane) {
#pragma unroll
  for (int k = 0; k < kPer; k++) {
    const int64_t i = base + lane + 32 * k;
    const bool v = i < end;
    c.t[k] = v ? __ldcs(A.arrival + i) : 0.0;
    c.x[k] = v ? __ldcs(A.input_len + i) : 0;
    c.y[k] = v ? __ldcs(A.output_len + i) : 0;
  }
}

// Fold one chunk [base, base + 32*kPer) (requests at or past `end` are
// padding; kFull: none are).  Lengths below 2^29 keep x^2, y^2, xy sums of
// one chunk inside 64 bits, so the 128-bit moments take one carry per chunk.
template <bool kFull>
__device__ __forceinline__ void fold_chunk(const arrow_stats_args_t& A, Acc& acc, Run& run, uint32_t* hist,
                                           const Chunk& c, int64_t base, int64_t end, int lane, double lo_d,
                                           double hi_d, double inv_b) {
  const double w = A.bucket_s;
  const uint32_t hist_sx = (uint32_t)__cvta_generic_to_shared(hist);
  const uint32_t hist_sy = hist_sx + 4u * kHistSpan;
  uint64_t qxx = 0, qyy = 0, qxy = 0;
  uint32_t big = 0;
  // Still in the run's bucket F?  For t >= 0 the bucket is trunc(t / w)
  // (see floordiv_fast), so t is in F iff F*w <= t < (F+1)*w, decided
  // exactly by the signs of two FMA residuals.  One vote for the whole
  // chunk: the common case (the chunk stays in the run) is branch-free.
  bool chunk_in = true;
#pragma unroll
  for (int k = 0; k < kPer; k++) {
    const bool v = kFull || base + lane + 32 * k < end;
    const double t = c.t[k];
    chunk_in = chunk_in && (!v || (fma(-run.f, w, t) >= 0.0 && fma(-run.f1, w, t) < 0.0));
  }
  chunk_in = __all_sync(FULL, chunk_in);
  if (kFull) {
    // arrival extremes as a tree (arrivals are never NaN; a +-0 tie may keep
    // either zero, only the duration max - min is used)
    double lo[kPer], hi[kPer];
#pragma unroll
    for (int k = 0; k < kPer; k++) lo[k] = hi[k] = c.t[k];
#pragma unroll
    for (int d = 1; d < kPer; d *= 2)
#pragma unroll
      for (int k = 0; k + d < kPer; k += 2 * d) {
        lo[k] = fmin(lo[k], lo[k + d]);
        hi[k] = fmax(hi[k], hi[k + d]);
      }
    acc.tmin = fmin(lo[0], acc.tmin);
    acc.tmax = fmax(hi[0], acc.tmax);
  }
#pragma unroll
  for (int k = 0; k < kPer; k++) {
    const bool v = kFull || base + lane + 32 * k < end;
    const double t = c.t[k];
    const int32_t x = c.x[k], y = c.y[k];
    if (chunk_in || __all_sync(FULL, !v || (fma(-run.f, w, t) >= 0.0 && fma(-run.f1, w, t) < 0.0))) {
      run.c += v ? 1u : 0u;
      run.x += (uint32_t)x;  // 0 on padding lanes
      run.y += (uint32_t)y;
    } else {
      bool ok;
      double f = floordiv_fast(t, w, inv_b, ok);
      if (v && !ok) f = py_floordiv(t, w);
      const bool inwin = f >= lo_d && f < hi_d;
      const double f0 = __shfl_sync(FULL, f, 0);
      if (__all_sync(FULL, !v || (ok && inwin && f == f0))) {
        // the whole slice is in one new bucket: restart the run there
        run.flush(A, acc, lo_d, lane);
        run.f = f0;
        run.f1 = f0 + 1.0;
        run.c = v ? 1u : 0u;
        run.x = (uint32_t)x;
        run.y = (uint32_t)y;
      } else {
        const int64_t b = (v && inwin) ? (int64_t)(f - lo_d) : -1;
        if (v && !inwin) acc.oow++;
        bucket_add(A, acc, b, x, y, lane);
      }
    }
    if (v) {
      if (!kFull) {
        acc.tmin = fmin(t, acc.tmin);
        acc.tmax = fmax(t, acc.tmax);
      }
      // predicated shared-memory reductions on precomputed shared-window
      // addresses (lengths outside 1..kBins are counted on the host as
      // n - sum(bins))
      hist_inc(hist_sx, x);
      hist_inc(hist_sy, y);
    }
    const uint64_t ux = (uint32_t)x, uy = (uint32_t)y;
    big |= (uint32_t)x | (uint32_t)y;
    qxx += ux * ux;
    qyy += uy * uy;
    qxy += ux * uy;
  }
  if (big < (1u << 29)) {
    acc.pxx += qxx;
    acc.pyy += qyy;
    acc.pxy += qxy;
    if (++acc.pn == 32 / kPer) acc.flush_pending();  // 32/kPer chunks of < kPer * 2^58 stay below 2^63
  } else {  // huge lengths: redo this chunk's moments with a carry per term
#pragma unroll
    for (int k = 0; k < kPer; k++) {
      const uint64_t ux = (uint32_t)c.x[k], uy = (uint32_t)c.y[k];
      acc.sxx.add(ux * ux);
      acc.syy.add(uy * uy);
      acc.sxy.add(ux * uy);
    }
  }
}

__device__ __forceinline__ void fold(const arrow_stats_args_t& A, Acc& acc, Run& run, uint32_t* hist,
                                     const Chunk& c, int64_t base, int64_t end, int lane, double lo_d, double hi_d,
                                     double inv_b) {
  if (base + kChunk <= end)
    fold_chunk<true>(A, acc, run, hist, c, base, end, lane, lo_d, hi_d, inv_b);
  else
    fold_chunk<false>(A, acc, run, hist, c, base, end, lane, lo_d, hi_d, inv_b);
}

// ---- TMA bulk-copy pipeline (cp.async.bulk + mbarrier), one ring per warp ----

#ifndef ARROW_STATS_STAGES
#define ARROW_STATS_STAGES 3
#endif
constexpr int kStages = ARROW_STATS_STAGES;
struct Stage {  // one chunk of the SoA trace, as it sits in HBM
  double t[kChunk];
  int32_t x[kChunk], y[kChunk];
};
constexpr uint32_t kStageBytes = sizeof(Stage);
static_assert(kStageBytes == 16 * kChunk, "stage = 16 B per request");
constexpr size_t kHistBytes = kHistWords * sizeof(uint32_t);
constexpr size_t kSmemBytes = kHistBytes + (size_t)kWarps * kStages * kStageBytes;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Arm the stage's barrier for 16 B/request and start its three bulk copies.
__device__ __forceinline__ void issue_stage(const arrow_stats_args_t& A, Stage* st, uint64_t* bar, int64_t base) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(kStageBytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(st->t)),
      "l"(A.arrival + base), "r"((uint32_t)(kChunk * 8)), "r"(smem_u32(bar))
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(st->x)),
      "l"(A.input_len + base), "r"((uint32_t)(kChunk * 4)), "r"(smem_u32(bar))
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(st->y)),
      "l"(A.output_len + base), "r"((uint32_t)(kChunk * 4)), "r"(smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(kStatsThreads, 1) arrow_stats_kernel(const arrow_stats_args_t A) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint32_t* hist = (uint32_t*)smem_raw;  // [2][kHistSpan]
  __shared__ Acc red[kWarps];
  __shared__ uint64_t bars[kWarps][kStages];
  for (int i = threadIdx.x; i < kHistWords; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  Acc acc;
  acc.init();
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  Run run{nan, nan, 0, 0, 0};
  const double lo_d = (double)A.bucket_lo;
  const double hi_d = lo_d + (double)A.n_buckets;  // exclusive
  const double inv_b = 1.0 / A.bucket_s;
  // warp w streams the contiguous range [w * per, (w + 1) * per)
  const int64_t n = A.n;
  const int64_t warps = (int64_t)gridDim.x * kWarps;
  const int64_t per = ((n + warps - 1) / warps + kChunk - 1) / kChunk * kChunk;
  const int64_t w = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t begin = w * per;
  const int64_t end = min(n, begin + per);
  const bool aligned = (((uintptr_t)A.arrival | (uintptr_t)A.input_len | (uintptr_t)A.output_len) & 15) == 0;
  if (aligned) {
    // Every full chunk of the warp's range streams HBM -> shared memory by
    // TMA bulk copies through a kStages-deep ring (one elected lane issues,
    // the mbarrier's transaction count says when the 16 B/request landed),
    // so ~kStages chunks per warp are in flight while the lanes fold; only
    // a partial last chunk is loaded through registers.
    Stage* ring = (Stage*)(smem_raw + kHistBytes) + warp * kStages;
    uint64_t* bar = bars[warp];
    const int64_t nfull = (end > begin) ? (end - begin) / kChunk : 0;
    if (lane == 0) {
      for (int q = 0; q < kStages; q++) mbar_init(&bar[q]);
      asm volatile("fence.mbarrier_init.release.cluster;\n fence.proxy.async.shared::cta;" ::: "memory");
      for (int q = 0; q < kStages && q < nfull; q++) issue_stage(A, &ring[q], &bar[q], begin + (int64_t)q * kChunk);
    }
    __syncwarp();
    int q = 0;             // stage of chunk j
    uint32_t parity = 0;   // phase of that stage's barrier
    for (int64_t j = 0; j < nfull; j++) {
      while (!mbar_try_wait(&bar[q], parity)) {
      }
      Chunk c;
#pragma unroll
      for (int k = 0; k < kPer; k++) {
        c.t[k] = ring[q].t[lane + 32 * k];
        c.x[k] = ring[q].x[lane + 32 * k];
        c.y[k] = ring[q].y[lane + 32 * k];
      }
      __syncwarp();  // every lane has read the stage before it is refilled
      if (lane == 0 && j + kStages < nfull) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_stage(A, &ring[q], &bar[q], begin + (j + kStages) * kChunk);
      }
      fold_chunk<true>(A, acc, run, hist, c, begin + j * kChunk, end, lane, lo_d, hi_d, inv_b);
      if (++q == kStages) {
        q = 0;
        parity ^= 1u;
      }
    }
    const int64_t tail = begin + nfull * kChunk;
    if (tail < end) {
      Chunk c;
      load_chunk(A, c, tail, end, lane);
      fold_chunk<false>(A, acc, run, hist, c, tail, end, lane, lo_d, hi_d, inv_b);
    }
  } else {
    // unaligned views: register double buffering (the next chunk's loads
    // are in flight while this one is folded)
    Chunk c0, c1;
    int64_t base = begin;
    if (base < end) load_chunk(A, c0, base, end, lane);
    while (base < end) {
      const int64_t b1 = base + kChunk;
      if (b1 < end) load_chunk(A, c1, b1, end, lane);
      fold(A, acc, run, hist, c0, base, end, lane, lo_d, hi_d, inv_b);
      if (b1 >= end) break;
      const int64_t b2 = b1 + kChunk;
      if (b2 < end) load_chunk(A, c0, b2, end, lane);
      fold(A, acc, run, hist, c1, b1, end, lane, lo_d, hi_d, inv_b);
      base = b2;
    }
  }
  run.flush(A, acc, lo_d, lane);
  acc.flush_pending();
  warp_merge(acc);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) {
    const uint32_t hx = hist[1 + i], hy = hist[kHistSpan + 1 + i];
    if (hx) atomicAdd(&A.hist_x[i], hx);
    if (hy) atomicAdd(&A.hist_y[i], hy);
  }
  if (threadIdx.x == 0) {
    Acc a = red[0];
    for (int q = 1; q < kWarps; q++) a.merge(red[q]);
    arrow_stats_partial_t p;
    p.min_arrival = a.count ? a.tmin : __longlong_as_double(0x7ff8000000000000ll);
    p.max_arrival = a.count ? a.tmax : __longlong_as_double(0x7ff8000000000000ll);
    p.count = a.count;
    p.sum_x = a.sx;
    p.sum_y = a.sy;
    p.sxx_lo = a.sxx.lo;
    p.sxx_hi = a.sxx.hi;
    p.syy_lo = a.syy.lo;
    p.syy_hi = a.syy.hi;
    p.sxy_lo = a.sxy.lo;
    p.sxy_hi = a.sxy.hi;
    p.out_of_window = a.oow;
    A.partials[blockIdx.x] = p;
  }
}

__global__ void arrow_stats_hist_kernel(const int32_t* __restrict__ values, int64_t n, int64_t lo, int64_t hi,
                                        int32_t shift, uint32_t* __restrict__ bins) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t v = __ldcs(values + i);
    if (v >= lo && v < hi) atomicAdd(&bins[(v - lo) >> shift], 1u);
  }
}

int sm_count() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 1;
  return sms > 0 ? sms : 1;
}

}  // namespace

extern "C" {

int arrow_stats_grid(int64_t n, int32_t* n_partials) {
  const int64_t chunks = (n + kPer * kStatsThreads - 1) / (kPer * kStatsThreads);
  const int64_t g = chunks < sm_count() ? chunks : sm_count();
  *n_partials = (int32_t)(g < 1 ? 1 : g);
  return 0;
}

int arrow_stats_run(const arrow_stats_args_t* a, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const size_t smem = kSmemBytes;
  cudaError_t e = cudaFuncSetAttribute(arrow_stats_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  if (a->n_buckets > 0) {
    const size_t nb = (size_t)a->n_buckets * sizeof(int64_t);
    if ((e = cudaMemsetAsync(a->bucket_requests, 0, nb, s)) != cudaSuccess) return (int)e;
    if ((e = cudaMemsetAsync(a->bucket_input, 0, nb, s)) != cudaSuccess) return (int)e;
    if ((e = cudaMemsetAsync(a->bucket_output, 0, nb, s)) != cudaSuccess) return (int)e;
  }
  if ((e = cudaMemsetAsync(a->hist_x, 0, kBins * sizeof(uint32_t), s)) != cudaSuccess) return (int)e;
  if ((e = cudaMemsetAsync(a->hist_y, 0, kBins * sizeof(uint32_t), s)) != cudaSuccess) return (int)e;
  if (a->n_partials < 1) return (int)cudaErrorInvalidValue;
  arrow_stats_kernel<<<a->n_partials, kStatsThreads, smem, s>>>(*a);
  return (int)cudaGetLastError();
}

int arrow_stats_hist(const int32_t* values, int64_t n, int64_t lo, int64_t hi, int32_t shift, uint32_t* bins,
                     int64_t n_bins, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(bins, 0, (size_t)n_bins * sizeof(uint32_t), s);
  if (e != cudaSuccess) return (int)e;
  if (n <= 0) return 0;
  const int blocks = 4 * sm_count();
  arrow_stats_hist_kernel<<<blocks, 512, 0, s>>>(values, n, lo, hi, shift, bins);
  return (int)cudaGetLastError();
}

int arrow_stats_layout(int64_t* out, int cap) {
  int64_t v[64];
  int n = 0;
#define SZ(T) v[n++] = (int64_t)sizeof(T)
#define OFF(T, f) v[n++] = (int64_t)offsetof(T, f)
  SZ(arrow_stats_partial_t);
  SZ(arrow_stats_args_t);
  OFF(arrow_stats_partial_t, min_arrival);
  OFF(arrow_stats_partial_t, max_arrival);
  OFF(arrow_stats_partial_t, count);
  OFF(arrow_stats_partial_t, sum_x);
  OFF(arrow_stats_partial_t, sum_y);
  OFF(arrow_stats_partial_t, sxx_lo);
  OFF(arrow_stats_partial_t, sxx_hi);
  OFF(arrow_stats_partial_t, syy_lo);
  OFF(arrow_stats_partial_t, syy_hi);
  OFF(arrow_stats_partial_t, sxy_lo);
  OFF(arrow_stats_partial_t, sxy_hi);
  OFF(arrow_stats_partial_t, out_of_window);
  OFF(arrow_stats_args_t, arrival);
  OFF(arrow_stats_args_t, input_len);
  OFF(arrow_stats_args_t, output_len);
  OFF(arrow_stats_args_t, n);
  OFF(arrow_stats_args_t, bucket_s);
  OFF(arrow_stats_args_t, bucket_lo);
  OFF(arrow_stats_args_t, n_buckets);
  OFF(arrow_stats_args_t, bucket_requests);
  OFF(arrow_stats_args_t, bucket_input);
  OFF(arrow_stats_args_t, bucket_output);
  OFF(arrow_stats_args_t, hist_x);
  OFF(arrow_stats_args_t, hist_y);
  OFF(arrow_stats_args_t, partials);
  OFF(arrow_stats_args_t, n_partials);
  OFF(arrow_stats_args_t, reserved);
#undef SZ
#undef OFF
  for (int i = 0; i < n && i < cap; i++) out[i] = v[i];
  return n;
}

}  // extern "C"
