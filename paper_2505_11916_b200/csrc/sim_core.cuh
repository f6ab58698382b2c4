// sim_core.cuh — one Arrow scheduling simulation per warp.
//
// Semantics are those of the reference discrete-event simulator (pdsim,
// /root/reference/pkg/src/pdsim); the data layout is B200-first:
//
//  * Instances map to lanes (instance i -> lane i % 32, register slot
//    i / 32).  Each lane keeps its instances' hot state in registers: KV
//    counters, incrementally maintained growth / running-token sums
//    (instance.py:159-173, 292-302 recomputed O(residents) per call in the
//    reference), the pending batch summary and ring cursors.
//  * Queues are per-instance rings in the slot's global workspace (L2
//    resident): waiting prefills carry their cached predictor term so the
//    predicted-delay fold (instance.py:304-321) streams independent loads;
//    waiting decodes and migrations are FIFO rings; running decodes are an
//    unordered array keyed by their finishing iteration (every running
//    decode is in every batch, instance.py:187-191 with the decode cap
//    invariant), so an iteration costs O(1) unless a decode finishes.
//  * The global event order (time, kind, seq) of the reference heap
//    (engine.py:39-45, 164-166) is reproduced exactly: every lane offers
//    its instances' pending ITERATION/MIGRATION completions, lane 0 the
//    arrival cursor, the PREFILL_COMPLETE FIFO head and the monitor tick,
//    and a three-step redux.sync argmin picks the next event.
//  * Scheduler decisions (scheduler.py:151-335) are warp argmins with
//    pool-insertion-order tie breaks; pool membership is an insertion
//    position per instance (pools.py:42-85).
//  * All floating point is IEEE double without contraction (built with
//    -fmad=false / -ffp-contract=off), in the reference's expression order;
//    Python's sum() is reproduced with CPython 3.12's Neumaier loop.
#pragma once

#include <math.h>
#include <stdint.h>
#include <string.h>

#include "arrow_sim.h"
#include "warp.cuh"

// Test-only mutants (host emulator build with -DARROW_MUTANTS, selected by
// the ARROW_MUTANT environment variable): tests prove that the tie fixture
// and the audit build can tell them from the shipped source.
#if !defined(__CUDA_ARCH__) && defined(ARROW_MUTANTS)
#include <stdlib.h>
#include <string.h>
#define MUTANT(name) (getenv("ARROW_MUTANT") != nullptr && strcmp(getenv("ARROW_MUTANT"), name) == 0)
#else
#define MUTANT(name) false
#endif

#if !defined(__CUDA_ARCH__) && defined(ARROW_EMU_TRACE)
#include <stdio.h>
#include <stdlib.h>
#define ATRACE(...)                                    \
  do {                                                 \
    if (getenv("ARROW_EMU_TRACE")) fprintf(stderr, __VA_ARGS__); \
  } while (0)
#else
#define ATRACE(...) \
  do {              \
  } while (0)
#endif

#if defined(ARROW_PROF) && defined(__CUDACC__)
#define ARROW_PROF_MAX 4096
__device__ int64_t arrow_prof_cycles[ARROW_PROF_MAX * 32];
#endif

namespace arrow {

enum { EV_MIG = 0, EV_ITER = 1, EV_PREFILL = 2, EV_ARRIVAL = 3, EV_TICK = 4 };
enum { P_PREFILL = 0, P_DECODE = 1, P_P2D = 2, P_D2P = 3 };
static constexpr int MAX_INST = 64;
#ifndef ARROW_DELAY_SLACK
#define ARROW_DELAY_SLACK 0x1p-52  // per-term slack of the delay interval (tests widen it to force exact folds)
#endif
static constexpr uint32_t SEQ_LIMIT = 1u << 28;
#ifndef ARROW_BURST_POOL
#define ARROW_BURST_POOL 512
#endif
#ifndef ARROW_BURST_MAX
#define ARROW_BURST_MAX 128
#endif
static constexpr int BURST_POOL = ARROW_BURST_POOL;  // chain-burst event keys per warp (shared memory)
static constexpr int BURST_MAX = ARROW_BURST_MAX;    // events per instance per chain burst

// ---------------------------------------------------------------- layout --

struct SlotLayout {
  int64_t n_max, N_max, qcap, rcap, ecap;
  int64_t off_first, off_last, off_ttft, off_tpot, off_src;
  int64_t off_fifo_time, off_fifo_rid, off_fifo_src, off_fifo_seq;
  int64_t off_wp_term, off_wp_rid, off_wd_rid, off_mq_rid, off_run_rid, off_run_f, off_em;
  int64_t bytes;
};

AS_HD int64_t align256(int64_t x) { return (x + 255) & ~(int64_t)255; }

AS_HD SlotLayout make_layout(int64_t n_max, int64_t N_max, int64_t qcap, int64_t rcap, int64_t ecap) {
  SlotLayout L;
  L.n_max = n_max < 1 ? 1 : n_max;
  L.N_max = N_max;
  L.qcap = qcap < 1 ? 1 : qcap;
  L.rcap = rcap < 1 ? 1 : rcap;
  L.ecap = ecap < 2 ? 2 : ecap;
  int64_t o = 0;
  const int64_t n = L.n_max;
  L.off_first = o; o = align256(o + 8 * n);
  L.off_last = o; o = align256(o + 8 * n);
  L.off_ttft = o; o = align256(o + 8 * n);
  L.off_tpot = o; o = align256(o + 8 * n);
  L.off_fifo_time = o; o = align256(o + 8 * n);
  L.off_wp_term = o; o = align256(o + 8 * N_max * L.qcap);
  L.off_em = o; o = align256(o + 8 * N_max * L.ecap);
  L.off_src = o; o = align256(o + 4 * n);
  L.off_fifo_rid = o; o = align256(o + 4 * n);
  L.off_fifo_src = o; o = align256(o + 4 * n);
  L.off_fifo_seq = o; o = align256(o + 4 * n);
  L.off_wp_rid = o; o = align256(o + 4 * N_max * L.qcap);
  L.off_wd_rid = o; o = align256(o + 4 * N_max * L.qcap);
  L.off_mq_rid = o; o = align256(o + 4 * N_max * L.qcap);
  L.off_run_rid = o; o = align256(o + 4 * N_max * L.rcap);
  L.off_run_f = o; o = align256(o + 4 * N_max * L.rcap);
  L.bytes = o;
  return L;
}

struct SlotPtrs {
  double *first, *last, *ttft, *tpot, *fifo_time, *wp_term, *em;
  int *src, *fifo_rid, *fifo_src, *wp_rid, *wd_rid, *mq_rid, *run_rid, *run_f;
  uint32_t* fifo_seq;
};

AS_HD SlotPtrs slot_ptrs(char* base, const SlotLayout& L) {
  SlotPtrs p;
  p.first = (double*)(base + L.off_first);
  p.last = (double*)(base + L.off_last);
  p.ttft = (double*)(base + L.off_ttft);
  p.tpot = (double*)(base + L.off_tpot);
  p.fifo_time = (double*)(base + L.off_fifo_time);
  p.wp_term = (double*)(base + L.off_wp_term);
  p.em = (double*)(base + L.off_em);
  p.src = (int*)(base + L.off_src);
  p.fifo_rid = (int*)(base + L.off_fifo_rid);
  p.fifo_src = (int*)(base + L.off_fifo_src);
  p.fifo_seq = (uint32_t*)(base + L.off_fifo_seq);
  p.wp_rid = (int*)(base + L.off_wp_rid);
  p.wd_rid = (int*)(base + L.off_wd_rid);
  p.mq_rid = (int*)(base + L.off_mq_rid);
  p.run_rid = (int*)(base + L.off_run_rid);
  p.run_f = (int*)(base + L.off_run_f);
  return p;
}

// ------------------------------------------------------------ state -----

// Warp-uniform scenario state (shared memory, one writer at a time,
// published with a warp sync).  engine.py:157-162, scheduler.py:82-85.
struct Uniform {
  double now;
  double tick_time;
  double breach;
  double next_arrival;
  double stall_time;
  double tmp_d;
  int64_t esp;
  int64_t n_events, n_iters, n_ticks, n_snap, n_dec;
  int64_t rr_p, rr_d;
  int64_t n_rounds, n_serial, n_bursts;
  int64_t cyc_serial, cyc_round, cyc_burst;   // profiling: SM cycles by step kind
  int64_t cyc_kind[32];                       // ARROW_PROF: serial cycles by event kind, rescan, selection/execution
  uint64_t hash;
  uint32_t seq, tick_seq;
  int a;
  int completed;
  int tick_active;
  int fifo_head, fifo_count;
  int status, overflow;
  int n_flips;
  int pool_n[4];
  int tmp_i[4];
};

struct WarpSmem {
  arrow_scenario_t sc;
  Uniform u;
  int16_t pool_of[MAX_INST];
  int16_t pos_of[MAX_INST];
  int list[MAX_INST];
  double vals[MAX_INST];
  int valid[MAX_INST];
  int hist[256];
  uint64_t blist[BURST_POOL];    // chain-burst event keys, one segment per instance
  int bcount[MAX_INST];          // events each instance ran in the current burst
  int boff[MAX_INST];            // its segment in blist
  int bhead[MAX_INST];           // merge cursor (tie fallback)
  int blast[MAX_INST];           // its last event pushed a successor
  uint32_t bseq[MAX_INST];       // sequence of its head / final pending push
  uint64_t bfinal[MAX_INST];     // key of its final pushing event (~0: none)
  int btie;
#ifdef ARROW_AUDIT
  int aud_parked_kv[MAX_INST];   // audit: KV parked on each instance, recounted from the queues
  int aud_parked_n[MAX_INST];
#endif
};

// Registers of one instance on its owner lane (instance.py:78-92, reshaped).
struct Inst {
  int id;                       // -1: unused slot
  int busy;
  double busy_until;
  uint32_t iter_seq;
  int mig_active, mig_rid;
  double mig_finish;
  uint32_t mig_seq;
  int kv_used, kv_reserved;
  int committed;                // sum over running decodes of out - 1 - generated
  int wgrowth;                  // sum over waiting decodes of out - 1
  int rtok;                     // running_tokens(): prompt + generated over resident decodes
  int R;                        // running decodes
  int min_f;                    // smallest finishing iteration among running decodes
  int it;                       // iterations begun
  int pb_ndec, pb_rp_chunk, pb_k, pb_last_chunk, pb_last_comp, pb_ded;
  int rp_rid, rp_done;          // the (at most one) partially prefilled running prompt
  int wp_h, wp_c, wd_h, wd_c, mq_h, mq_c, em_h, em_c;
  int parked;
  int min_f_cnt;                // running decodes finishing at min_f
  int pb_pc, pb_emit;           // pending iteration pushes a PREFILL_COMPLETE / emits a token
  int pb_rel;                   // KV released by single-token requests completing in the pending iteration
  int pb_rp_left;               // the running partial prompt survives the pending iteration
  int held_min;                 // KV held by the running decodes finishing at min_f
  int mq_need;                  // KV need of the migration queue head (valid when mq_c > 0)
  double em_first, em_last;     // oldest / newest time in the emission ring (valid when em_c > 0)
  int cq;                       // cached: pending iteration is quiet
  uint64_t ck;                  // cached: order key of busy_until
  double dly;                   // predicted_prefill_delay at the current event (exact iff dexact)
  double dlo, dhi;              // interval certainly holding the exact predicted_prefill_delay
  int dexact;                   // dly is the exact left fold
  int pool;                     // register copy of sm->pool_of[id] (owner lane)
  double ws_hi, ws_lo;          // waiting-prefill terms: double-double running sum ...
  double ws_max;                // ... and the largest |term| since the queue was last empty
};

AS_HD uint64_t dbits(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
}

// Order-preserving map double -> uint64 (-0.0 canonicalised to +0.0, as
// Python's `<` treats them equal).
AS_HD uint64_t okey(double x) {
  uint64_t u = dbits(x + 0.0);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// Order key of an event time.  Event times are >= +0.0 (arrivals are
// validated >= 0 and canonicalised on the host, core.py:47-48; every other
// time is t + a positive duration; the burst caps below are t + a positive
// span), so the key is the bit pattern with the sign bit set: one OR instead
// of okey's sign select and canonicalising add.
AS_HD uint64_t tkey(double t) { return dbits(t) | 0x8000000000000000ull; }

// Inverse of tkey (keys of event times, sign bit always set).
AS_HD double tkey_inv(uint64_t k) {
  const uint64_t u = k & 0x7fffffffffffffffull;
  double x;
  memcpy(&x, &u, 8);
  return x;
}

AS_HD double okey_inv(uint64_t k) {
  uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double x;
  memcpy(&x, &u, 8);
  return x;
}

AS_HD int ffs32(uint32_t m) {
#ifdef __CUDA_ARCH__
  return __ffs((int)m) - 1;
#else
  return m ? __builtin_ctz(m) : -1;
#endif
}

AS_HD int popc32(uint32_t m) {
#ifdef __CUDA_ARCH__
  return __popc(m);
#else
  return __builtin_popcount(m);
#endif
}

// cost_model.py:73-92, reference expression order
AS_HD double quad(double a2, double a1, double a0, int len) {
  double L = (double)len;
  return a2 * L * L + a1 * L + a0;
}

AS_HD int imin(int a, int b) { return a < b ? a : b; }

// min(BURST_POOL / n, BURST_MAX) for 1 <= n <= 64 without an integer
// division (a ~20-instruction sequence): POOL/n is an integer or at least 1/64
// away from one, far more than __fdividef's 2-ulp error (POOL <= 2^14), so
// floor(q + 1/1024) is exact.
AS_HD int burst_share(uint32_t n) {
  static_assert(BURST_POOL <= (1 << 14) && BURST_POOL % BURST_MAX == 0, "burst_share bounds");
  if (n <= (uint32_t)(BURST_POOL / BURST_MAX)) return BURST_MAX;
#ifdef __CUDA_ARCH__
  return __float2int_rz(__fdividef((float)BURST_POOL, (float)n) + 0x1p-10f);
#else
  return (int)(BURST_POOL / n);
#endif
}

// ------------------------------------------------------------- simulator --

#ifdef ARROW_PROF
#define PROF_CLOCK(var) const int64_t var = clock_now()
#define PROF_ADD(field, since)                           \
  do {                                                   \
    const int64_t _now = clock_now();                    \
    if (lane == 0) u().field += _now - (since);          \
  } while (0)
#define PROF_MARK(slot, since)                              \
  do {                                                      \
    const int64_t _now = clock_now();                       \
    if (lane == 0) u().cyc_kind[slot] += _now - (since);    \
  } while (0)
#else
#define PROF_CLOCK(var) \
  do {                  \
  } while (0)
#define PROF_ADD(field, since) \
  do {                         \
  } while (0)
#define PROF_MARK(slot, since) \
  do {                         \
  } while (0)
#endif

// COMPACT (the occupancy build): code size over instruction count.  With 12
// warps per SM at unrelated points of the event loop the hot code does not
// fit the instruction caches (C5 ncu: 78 % of stall samples "no
// instruction"), so repeated call sites are folded into non-unrolled loops.
// The latency build (1-2 warps per SM) keeps them unrolled.
#define HAVE_OM (!LEAN && have_om)

#if defined(__CUDA_ARCH__)
#define AS_NOINL __noinline__
#else
#define AS_NOINL __attribute__((noinline))
#endif

// The waiting-prefill part of predicted_prefill_delay (instance.py:318-321):
// d += term for each waiting prompt, in queue order (a left fold), from the
// ring of cached predictor terms.  Out of line: the exact fold is the rare
// fallback of the delay intervals, and inlined it cost one unrolled copy per
// call site.
AS_NOINL AS_HD double delay_fold(double d, const double* t, int h, int c, int cap) {
  int j = 0;
  for (; j + 4 <= c; j += 4) {
    const int a = h + j >= cap ? h + j - cap : h + j;
    const int b = a + 1 >= cap ? a + 1 - cap : a + 1;
    const int e = b + 1 >= cap ? b + 1 - cap : b + 1;
    const int f = e + 1 >= cap ? e + 1 - cap : e + 1;
    const double t0 = t[a], t1 = t[b], t2 = t[e], t3 = t[f];
    d += t0;
    d += t1;
    d += t2;
    d += t3;
  }
  for (; j < c; j++) d += t[h + j >= cap ? h + j - cap : h + j];
  return d;
}

// avg_token_interval's window pruning and mean (instance.py:323-329) on one
// instance's emission ring, out of line: inlined, its gallop, binary search
// and IEEE fp64 division cost one copy per call site (emit, the pool mean at
// its two callers, the decode admission test).  State goes in and out by
// value so the call keeps the simulator in registers.
struct EmWin {
  double first;   // em_first after pruning
  double val;     // the interval (valid when ok)
  int h, c;       // ring head / count after pruning
  int ok;
};

// PROBE: start the search at the interpolated offset (emission times are
// close to evenly spaced; only the search start depends on it, never the
// result).  Used by the two-instances-per-lane build (C4 -4.5 %); the
// one-instance builds keep exactly the plain gallop (C5 +0.7 % with it).
template <bool PROBE>
AS_NOINL AS_HD EmWin em_window(const double* e, int h, int c, double first, double last, double lo, int cap) {
  if (c > 0 && first < lo) {
    // gallop from the head, then binary search: the first offset with t >= lo
    int a = 0, b = 0, step = 1;
    double vb = 0.0;
    if (PROBE && c > 16 && last >= lo) {
#ifdef __CUDA_ARCH__
      int g = __float2int_rz(__fdividef((float)(lo - first), (float)(last - first)) * (float)(c - 1));
#else
      int g = (int)((float)(lo - first) / (float)(last - first) * (float)(c - 1));
#endif
      g = g < 1 ? 1 : (g > c - 1 ? c - 1 : g);
      const int rg = h + g >= cap ? h + g - cap : h + g;
      const double vg = e[rg];
      if (vg < lo) {
        a = g;                 // gallop upward from the probe
      } else {
        const int g2 = g >> 1; // one halving step, then the binary search
        const int r2 = h + g2 >= cap ? h + g2 - cap : h + g2;
        const double v2 = e[r2];
        if (v2 < lo) {
          a = g2;
          b = g;
          vb = vg;
        } else {
          b = g2;
          vb = v2;
        }
        goto search;           // bracketed: no gallop
      }
    }
    for (;;) {
      b = a + step;
      if (b >= c) {
        b = c;
        break;
      }
      const int rb = h + b >= cap ? h + b - cap : h + b;
      vb = e[rb];
      if (vb >= lo) break;
      a = b;
      step <<= 1;
    }
  search:
    while (b - a > 1) {
      const int mid = (a + b) >> 1;
      const int rm = h + mid >= cap ? h + mid - cap : h + mid;
      const double vm = e[rm];
      if (vm < lo) {
        a = mid;
      } else {
        b = mid;
        vb = vm;
      }
    }
    h = h + b >= cap ? h + b - cap : h + b;
    c -= b;
    if (c > 0) first = vb;
  }
  EmWin r;
  r.first = first;
  r.h = h;
  r.c = c;
  r.ok = c >= 2;
  r.val = r.ok ? (last - first) / (double)(c - 1) : 0.0;
  return r;
}

// _pool_mean_interval's ordered Neumaier sum (scheduler.py:124-134) over the
// collected intervals, divided by their count; out of line (two callers).
// ok = 0 when no interval is valid.
struct MeanOut {
  double v;
  int ok;
};

AS_NOINL AS_HD MeanOut pool_mean_sum(const double* vals, const int* valid, int m) {
  double f = 0.0, c = 0.0;
  int cnt = 0;
  for (int j = 0; j < m; j++) {
    if (!valid[j]) continue;
    double x = vals[j];
    if (cnt == 0) {
      f = 0.0 + x;
    } else {
      double t = f + x;
      if (fabs(f) >= fabs(x))
        c += (f - t) + x;
      else
        c += (x - t) + f;
      f = t;
    }
    cnt++;
  }
  MeanOut r;
  r.ok = cnt > 0;
  if (c != 0.0 && isfinite(c)) f += c;
  r.v = r.ok ? f / (double)cnt : 0.0;
  return r;
}

// First error wins (status codes of include/arrow_sim.h).  A free function
// taking the shared-memory state by pointer, so the out-of-line call does
// not force the simulator object out of registers.
AS_NOINL AS_HD void status_set(Uniform* U, int s, int ovf) {
  if (U->status == ARROW_OK) {
    U->status = s;
    if (ovf != ARROW_OVF_NONE) U->overflow = ovf;
  }
}

// LEAN: the batch requests no optional outputs (a sweep: summaries only);
// every per-request / decision / snapshot / iteration-log write and its test
// compile out of the hot paths.
template <class W, int IPL, bool COMPACT = false, bool LEAN = false>
struct Sim {
  W w;
  WarpSmem* sm;
  const arrow_batch_t* B;
  SlotLayout L;
  SlotPtrs p;
  int lane;
  int sid;
  const double* arr;
  const int32_t* inl;
  const int32_t* outl;
  arrow_outmap_t om;
  bool have_om;                 // read through HAVE_OM
  Inst st[IPL];

  static constexpr int WD = W::WIDTH;

  AS_HD const arrow_scenario_t& sc() const { return sm->sc; }
  AS_HD Uniform& u() { return sm->u; }

  AS_HD static int lane_of(int id) { return id & (WD - 1); }

  // Run f(Inst&) on the owner lane of instance id, then publish.
  template <class F>
  AS_HD void owner(int id, F&& f) {
    if (lane == lane_of(id)) {
      if (IPL == 1 || id < WD)
        f(st[0]);
      else
        f(st[IPL - 1]);
    }
    w.sync();
  }

  template <class F>
  AS_HD void lane0(F&& f) {
    if (lane == 0) f();
    w.sync();
  }

  template <class G>
  AS_HD double bcast_d(int id, G g) {
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < IPL; k++)
      if (st[k].id == id) v = g(st[k]);
    return w.shfl(v, lane_of(id));
  }

  template <class G>
  AS_HD int bcast_i(int id, G g) {
    int v = 0;
#pragma unroll
    for (int k = 0; k < IPL; k++)
      if (st[k].id == id) v = g(st[k]);
    return w.shfl(v, lane_of(id));
  }

  // caller must be a single lane; out of line (error paths only)
  AS_HD void set_status(int s, int ovf = ARROW_OVF_NONE) { status_set(&sm->u, s, ovf); }

  // The 2^28 sequence budget (the order key packs kind << 28 | seq) is
  // checked once per step (serial bookkeeping, rounds, bursts, end of run),
  // not at every push: a run that exhausts it ends as BUFFER_OVERFLOW.
  AS_HD uint32_t next_seq() { return u().seq++; }

  // The 2^28 budget test on the per-step paths (lane 0).  The latency build
  // (!COMPACT) uses a branch-free form (selects and plain stores: no call and
  // no nested reconvergence region); the occupancy build keeps the call (the
  // branch-free form cost C5 2.4 % through code layout).  First error wins
  // either way, as in status_set().
  AS_HD void seq_check(uint32_t seq) {
    if (COMPACT) {
      if (seq >= SEQ_LIMIT) set_status(ARROW_BUFFER_OVERFLOW, ARROW_OVF_SEQ);
    } else {
      Uniform& U = u();
      const bool over = seq >= SEQ_LIMIT && U.status == ARROW_OK;
      const int st0 = U.status, ov0 = U.overflow;
      U.status = over ? ARROW_BUFFER_OVERFLOW : st0;
      U.overflow = over ? ARROW_OVF_SEQ : ov0;
    }
  }

  // ------------------------------------------------------ warp argmin --

  AS_HD int warp_argmin(uint64_t key, uint32_t tie, bool valid) {
    // each stage stops as soon as a single lane is left
    uint32_t b = w.ballot(valid);
    const uint32_t hi = w.min_u32(valid ? (uint32_t)(key >> 32) : ~0u);  // issued with the ballot
    if ((b & (b - 1)) == 0) return b ? ffs32(b) : -1;
    bool m = valid && (uint32_t)(key >> 32) == hi;
    b = w.ballot(m);
    if ((b & (b - 1)) == 0) return ffs32(b);
    const uint32_t lo = w.min_u32(m ? (uint32_t)key : ~0u);
    m = m && (uint32_t)key == lo;
    b = w.ballot(m);
    if ((b & (b - 1)) == 0) return ffs32(b);
    const uint32_t tt = w.min_u32(m ? tie : ~0u);
    m = m && tie == tt;
    return ffs32(w.ballot(m));
  }

  // First minimum over instances selected by kf (key, tie); returns the
  // instance id or -1 (scheduler.py:89-99: strict `<` in insertion order).
  template <class KF>
  AS_HD int argmin_inst(KF kf) {
    uint64_t bk = ~0ull;
    uint32_t bt = ~0u;
    int bid = -1;
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      if (st[k].id < 0) continue;
      uint64_t key;
      uint32_t tie;
      if (!kf(st[k], key, tie)) continue;
      if (bid < 0 || key < bk || (key == bk && tie < bt)) {
        bk = key;
        bt = tie;
        bid = st[k].id;
      }
    }
    int wl = warp_argmin(bk, bt, bid >= 0);
    if (wl < 0) return -1;
    return w.shfl(bid, wl);
  }

  AS_HD int pool_of(int id) const { return sm->pool_of[id]; }
  AS_HD int pos_of(int id) const { return sm->pos_of[id]; }

  // ---------------------------------------------------- global memory --

  AS_HD int* wp_rid(int id) { return p.wp_rid + (int64_t)id * L.qcap; }
  AS_HD double* wp_term(int id) { return p.wp_term + (int64_t)id * L.qcap; }
  AS_HD int* wd_rid(int id) { return p.wd_rid + (int64_t)id * L.qcap; }
  AS_HD int* mq_rid(int id) { return p.mq_rid + (int64_t)id * L.qcap; }
  AS_HD int* run_rid(int id) { return p.run_rid + (int64_t)id * L.rcap; }
  AS_HD int* run_f(int id) { return p.run_f + (int64_t)id * L.rcap; }
  AS_HD double* em(int id) { return p.em + (int64_t)id * L.ecap; }

  AS_HD int ring(int h, int j, int64_t cap) const {
    const int x = h + j;                  // h, j < cap <= 2^30
    return x >= (int)cap ? x - (int)cap : x;
  }

  // -------------------------------------------- instance-local (owner) --

  AS_HD bool has_prefill_work(const Inst& I) const { return I.rp_rid >= 0 || I.wp_c > 0; }
  AS_HD bool has_decode_work(const Inst& I) const { return I.mig_active || I.mq_c > 0 || I.R > 0 || I.wd_c > 0; }
  AS_HD bool startable(const Inst& I) const { return I.R > 0 || I.rp_rid >= 0 || I.wp_c > 0 || I.wd_c > 0; }

  // predicted_prefill_delay, instance.py:304-321 (left fold, same order)
  AS_HD double delay(const Inst& I, double now) {
    const arrow_scenario_t& s = sc();
    double d = 0.0;
    if (I.busy) {
      double x = I.busy_until - now;
      d += (0.0 > x) ? 0.0 : x;
    }
    if (I.rp_rid >= 0) d += quad(s.pred_a2, s.pred_a1, s.pred_a0, inl[I.rp_rid] - I.rp_done);
    return I.wp_c ? delay_fold(d, wp_term(I.id), I.wp_h, I.wp_c, (int)L.qcap) : d;
  }

  // Double-double accumulate (hi, lo) += t (Knuth two-sum; no contraction).
  AS_HD static void dd_add(double& hi, double& lo, double t) {
    const double s = hi + t;
    const double bb = s - hi;
    const double e = (hi - (s - bb)) + (t - bb) + lo;
    hi = s + e;
    lo = e - (hi - s);
  }

  // The exact delay is a left fold of up to n = wp_c + 2 terms; instead of
  // refolding a queue of up to hundreds of terms (a serially dependent chain
  // of double additions) for every dispatch, bracket it: the fold differs from
  // the real sum by at most (n - 1) u T (u = 2^-53, T = sum of |terms|), and
  // x0 + rp + (exact running sum of the waiting terms) by at most a few u T,
  // so [a - B, a + B] with B = (n + 8) 2^-52 T holds it.  Decisions that the
  // interval settles (argmin winner strictly below every other candidate, a
  // threshold test on the same side at both ends) are the reference's; the
  // rest fold exactly (delay()).  With no waiting prefills the fold is
  // x0 + rp itself and is exact.
  AS_HD void delay_interval(Inst& I, double now) {
    const arrow_scenario_t& s = sc();
    double x0 = 0.0, rp = 0.0;
    if (I.busy) {
      const double x = I.busy_until - now;
      x0 = (0.0 > x) ? 0.0 : x;
    }
    if (I.rp_rid >= 0) rp = quad(s.pred_a2, s.pred_a1, s.pred_a0, inl[I.rp_rid] - I.rp_done);
    if (I.wp_c == 0) {
      I.dly = I.dlo = I.dhi = (I.busy ? x0 : 0.0) + rp;  // the fold itself: 0.0 (+ x0) (+ rp)
      I.dexact = 1;
      return;
    }
    const double a = (x0 + rp) + (I.ws_hi + I.ws_lo);
    const double T = x0 + fabs(rp) + (double)I.wp_c * I.ws_max;
    const double B = (double)(I.wp_c + 10) * ARROW_DELAY_SLACK * T * (1.0 + 0x1p-30) + 0x1p-1000;
    I.dly = a;
    I.dlo = a - B;
    I.dhi = a + B;
    I.dexact = 0;
  }

  AS_HD void delay_exact(Inst& I, double now) {
    if (I.dexact) return;
    I.dly = I.dlo = I.dhi = delay(I, now);
    I.dexact = 1;
  }

  // avg_token_interval, instance.py:323-329: over emissions with
  // t >= now - window.  The ring holds this instance's emission times in
  // increasing order; entries older than any future query window are
  // dropped lazily (here, by binary search, and when the ring fills), which
  // is exact because query times never decrease.
  AS_HD bool interval(Inst& I, double now, double* out) {
    const EmWin r = em_window<(IPL == 2 || !COMPACT)>(em(I.id), I.em_h, I.em_c, I.em_first, I.em_last, now - sc().window,
                                          (int)L.ecap);
    I.em_h = r.h;
    I.em_c = r.c;
    I.em_first = r.first;
    *out = r.val;
    return r.ok != 0;
  }

  AS_HD void emit(Inst& I, double now) {
    double* e = em(I.id);
    if (I.em_c >= L.ecap) {
      double v;
      interval(I, now, &v);             // drops everything outside the window
      if (I.em_c >= L.ecap) {
        set_status(ARROW_BUFFER_OVERFLOW, ARROW_OVF_EMISSION);
        return;
      }
    }
    e[ring(I.em_h, I.em_c, L.ecap)] = now;
    if (I.em_c == 0) I.em_first = now;
    I.em_last = now;
    I.em_c++;
  }

  // advance_migrations, instance.py:126-146.  Returns true when a transfer
  // starts; the caller assigns its push sequence (engine.py:179-181).
  AS_HD bool start_mig(Inst& I, double now) {
    if (I.mig_active || I.mq_c == 0) return false;
    int rid = mq_rid(I.id)[I.mq_h];
    int need = inl[rid] + (outl[rid] - 1);
    int kvf = sc().kv_capacity - I.kv_used - I.kv_reserved - I.committed;
    if (kvf - I.wgrowth < need) return false;
    I.mq_h = I.mq_h + 1 == L.qcap ? 0 : I.mq_h + 1;
    I.mq_c--;
    if (I.mq_c > 0) {
      const int nr = mq_rid(I.id)[I.mq_h];
      I.mq_need = inl[nr] + (outl[nr] - 1);
    }
    I.kv_reserved += inl[rid] + (MUTANT("kv") ? 1 : 0);   // (mutant "kv": reservation off by one)
    I.mig_active = 1;
    I.mig_rid = rid;
    const arrow_scenario_t& s = sc();
    I.mig_finish = now + (s.base_latency + (double)((int64_t)inl[rid] * s.bytes_per_token) / s.bandwidth);
    return true;
  }

  // _kick + build_iteration_batch + begin_iteration (engine.py:170-177,
  // instance.py:175-252).  Returns true when an iteration starts; the caller
  // assigns its push sequence.  Also records whether the iteration will emit
  // a token and whether it will push a PREFILL_COMPLETE (for the parallel
  // rounds' quiet test).
  AS_HD bool kick(Inst& I, double now) {
    if (I.busy || !startable(I)) return false;
    const arrow_scenario_t& s = sc();
    const int budget = s.chunk_budget;
    const int dcap = imin(s.max_batch, budget);
    int kvf = s.kv_capacity - I.kv_used - I.kv_reserved - I.committed;
    if (I.R > dcap) {
      set_status(ARROW_INTERNAL);
      return false;
    }
    int nd = I.R, ad = 0;
    const int* wd = wd_rid(I.id);
    while (ad < I.wd_c && nd < dcap) {
      int rid = wd[ring(I.wd_h, ad, L.qcap)];
      int g = outl[rid] - 1;
      if (g > kvf) break;
      kvf -= g;
      nd++;
      ad++;
    }
    int rp_chunk = 0, k = 0, last_chunk = 0, last_comp = 0, ded = 0;
    int total = nd;
    int pc = 0;                 // completing prefills with output_len > 1
    int rel = 0;                // completing prefills with output_len == 1 (KV released)
    int done_pf = 0;            // completing prefills
    const int* wp = wp_rid(I.id);
    bool planned = false;
    if (nd == 0 && I.rp_rid < 0 && I.wp_c > 0) {
      int rid = wp[I.wp_h];
      int len = inl[rid];
      if (len <= budget && len <= kvf) {
        k = 1;
        last_chunk = len;
        last_comp = 1;
        ded = 1;
        total = len;
        planned = true;
        done_pf = 1;
        pc = outl[rid] > 1;
        rel = outl[rid] == 1 ? len : 0;
      }
    }
    if (!planned) {
      int left = budget - nd;
      bool stop = false;
      if (I.rp_rid >= 0) {
        if (left <= 0) {
          stop = true;
        } else {
          int rem = inl[I.rp_rid] - I.rp_done;
          int c = imin(imin(left, rem), kvf);
          if (c <= 0) {
            stop = true;
          } else {
            rp_chunk = c;
            left -= c;
            kvf -= c;
            total += c;
            if (c == rem) {
              done_pf++;
              pc |= outl[I.rp_rid] > 1;
              rel += outl[I.rp_rid] == 1 ? inl[I.rp_rid] : 0;
            }
          }
        }
      }
      while (!stop && k < I.wp_c) {
        if (left <= 0) break;
        int rid = wp[ring(I.wp_h, k, L.qcap)];
        int rem = inl[rid];
        int c = imin(imin(left, rem), kvf);
        if (c <= 0) break;
        k++;
        last_chunk = c;
        last_comp = c == rem;
        if (last_comp) {
          done_pf++;
          pc |= outl[rid] > 1;
          rel += outl[rid] == 1 ? rem : 0;
        }
        left -= c;
        kvf -= c;
        total += c;
      }
    }
    if (nd == 0 && rp_chunk == 0 && k == 0) return false;
    // begin_iteration
    const int cur = I.it++;
    if (ad > 0) {
      int* rr = run_rid(I.id);
      int* rf = run_f(I.id);
      int32_t* dit = (B->req_decode_iter && HAVE_OM && om.req_offset >= 0) ? B->req_decode_iter + om.req_offset
                                                                            : (int32_t*)0;
      for (int j = 0; j < ad; j++) {
        int rid = wd[ring(I.wd_h, j, L.qcap)];
        int g = outl[rid] - 1;
        int f = cur + g - 1;
        if (I.R >= L.rcap) {
          set_status(ARROW_BUFFER_OVERFLOW, ARROW_OVF_RUNNING);
          return false;
        }
        rr[I.R] = rid;
        rf[I.R] = f;
        I.R++;
        const int held = inl[rid] + g;
        if (f < I.min_f) {
          I.min_f = f;
          I.min_f_cnt = 1;
          I.held_min = held;
        } else if (f == I.min_f) {
          I.min_f_cnt++;
          I.held_min += held;
        }
        I.committed += g;
        I.wgrowth -= g;
        if (dit) dit[rid] = cur;
      }
      I.wd_h = ring(I.wd_h, ad, L.qcap);
      I.wd_c -= ad;
    }
    I.kv_used += total - nd;
    if (I.kv_used + I.kv_reserved > s.kv_capacity) set_status(ARROW_INTERNAL);
    I.pb_ndec = nd;
    I.pb_rp_chunk = rp_chunk;
    I.pb_k = k;
    I.pb_last_chunk = last_chunk;
    I.pb_last_comp = last_comp;
    I.pb_ded = ded;
    I.pb_pc = pc;
    I.pb_rel = rel;
    I.pb_rp_left = I.rp_rid >= 0 && !(rp_chunk > 0 && rp_chunk == inl[I.rp_rid] - I.rp_done);
    I.pb_emit = (nd + done_pf) > 0;
    double dur = ded ? quad(s.true_a2, s.true_a1, s.true_a0, last_chunk) : s.b1 * (double)total + s.b0;
    I.busy_until = now + dur;
    I.busy = 1;
    return true;
  }

  // A prompt finished prefill: first token, park its KV, then either the
  // single-token completion or a PREFILL_COMPLETE push (engine.py:212-218).
  // PREFILL_COMPLETE pushes only happen on the serial path.
  AS_HD void prefill_finished(Inst& I, int rid, double now, int& completed) {
    p.first[rid] = now;
    if (outl[rid] == 1) {
      I.kv_used -= inl[rid];      // release_parked, instance.py:120-122
      p.last[rid] = now;
      completed++;
    } else {
      I.parked++;
      int c = u().fifo_count;
      int slot = ring(u().fifo_head, c, L.n_max);
      p.fifo_rid[slot] = rid;
      p.fifo_src[slot] = I.id;
      p.fifo_time[slot] = now;
      p.fifo_seq[slot] = next_seq();
      u().fifo_count = c + 1;
    }
  }

  // ITERATION_COMPLETE for one instance: execute_iteration + the engine
  // handler (instance.py:254-288, engine.py:205-223).  Touches only this
  // instance's state and per-request outputs, except (SERIAL only) the
  // PREFILL_COMPLETE FIFO and the push sequence.  Adds finished requests to
  // `completed`; returns the drained-pool move (-1 none); sets `pushed` when
  // the next iteration started (non-SERIAL: lane-parallel rounds; the serial
  // path starts migrations and kicks in serial_tail()).
  AS_HD int iteration_complete(Inst& I, double now, int& completed, bool serial) {
    const int cur = I.it - 1;
    if (B->iterlog && HAVE_OM && om.iterlog_offset >= 0) {
      if (cur < om.iterlog_stride)
        B->iterlog[om.iterlog_offset + (int64_t)I.id * om.iterlog_stride + cur] = now;
      else if (u().overflow == ARROW_OVF_NONE)
        u().overflow = ARROW_OVF_ITERLOG;
    }
    const int nd = I.pb_ndec;
    int npf = 0;
    if (nd > 0) {
      I.kv_used += nd;
      I.committed -= nd;
      I.rtok += nd;
      if (I.min_f == cur) {
        int* rr = run_rid(I.id);
        int* rf = run_f(I.id);
        int m = 0x7fffffff, mc = 0, mh = 0;
        int j = 0;
        while (j < I.R) {
          int f = rf[j];
          if (f == cur) {
            int rid = rr[j];
            int held = inl[rid] + outl[rid] - 1;
            I.kv_used -= held;
            I.rtok -= held;
            p.last[rid] = now;
            completed++;
            I.R--;
            rr[j] = rr[I.R];
            rf[j] = rf[I.R];
          } else {
            const int hh = inl[rr[j]] + outl[rr[j]] - 1;
            if (f < m) {
              m = f;
              mc = 1;
              mh = hh;
            } else if (f == m) {
              mc++;
              mh += hh;
            }
            j++;
          }
        }
        I.min_f = m;
        I.min_f_cnt = mc;
        I.held_min = mh;
      }
    }
    if (I.pb_rp_chunk > 0) {
      I.rp_done += I.pb_rp_chunk;
      if (I.rp_done == inl[I.rp_rid]) {
        int rid = I.rp_rid;
        I.rp_rid = -1;
        npf++;
        prefill_finished(I, rid, now, completed);
      }
    }
    if (I.pb_k > 0) {
      const int* wp = wp_rid(I.id);
      const double* wt = wp_term(I.id);
      for (int j = 0; j < I.pb_k; j++) {
        int rid = wp[ring(I.wp_h, j, L.qcap)];
        dd_add(I.ws_hi, I.ws_lo, -wt[ring(I.wp_h, j, L.qcap)]);
        if (j < I.pb_k - 1 || I.pb_last_comp) {
          npf++;
          prefill_finished(I, rid, now, completed);
        } else {
          I.rp_rid = rid;
          I.rp_done = I.pb_last_chunk;
        }
      }
      I.wp_h = ring(I.wp_h, I.pb_k, L.qcap);
      I.wp_c -= I.pb_k;
      if (I.wp_c == 0) I.ws_hi = I.ws_lo = I.ws_max = 0.0;
    }
    I.busy = 0;
    I.pb_ndec = I.pb_rp_chunk = I.pb_k = I.pb_last_chunk = I.pb_last_comp = I.pb_ded = 0;
    if (nd + npf > 0) emit(I, now);
    // _check_drained (engine.py:183-192): decided here, applied by the warp
    int dst = -1;
    int pk = I.pool;
    if (pk == P_P2D && !has_prefill_work(I))
      dst = P_DECODE;
    else if (pk == P_D2P && !has_decode_work(I))
      dst = P_PREFILL;
    if (serial && nd + npf > 0) u().esp = 0;
    // _start_migrations (serial path) and _kick follow in simulate(): one
    // shared kick site for the serial and the lane-parallel paths
    return dst;
  }

  // ------------------------------------------------------ decisions ----

  AS_HD void log_decision(double now, int kind, int rid, int inst, int code) {
    // lane 0 only
    Uniform& U = u();
    uint64_t h = U.hash;
    h = (h ^ dbits(now)) * 1099511628211ull;
    uint64_t w2 = (uint64_t)kind | ((uint64_t)code << 8) | ((uint64_t)(uint16_t)inst << 16) |
                  ((uint64_t)(uint32_t)rid << 32);
    h = (h ^ w2) * 1099511628211ull;
    U.hash = h;
    if (B->decisions && HAVE_OM && om.decision_offset >= 0) {
      if (U.n_dec < om.decision_capacity) {
        arrow_decision_t* d = B->decisions + om.decision_offset + U.n_dec;
        d->time = now;
        d->request = rid;
        d->instance = (int16_t)inst;
        d->kind = (uint8_t)kind;
        d->code = (uint8_t)code;
      } else if (U.overflow == ARROW_OVF_NONE) {
        U.overflow = ARROW_OVF_DECISIONS;
      }
    }
    U.n_dec++;
  }

  AS_HD void log_dispatch(double now, int kind, int rid, int inst, int branch) {
    lane0([&] {
      log_decision(now, kind, rid, inst, branch);
      if (HAVE_OM && om.req_offset >= 0) {
        int32_t* out = kind == ARROW_DEC_PREFILL_DISPATCH ? B->req_prefill : B->req_decode;
        if (out) out[om.req_offset + rid] = inst | (branch << 16);
      }
    });
  }

  // PoolSet._move (pools.py:76-85) + the flip record (scheduler.py:109-119).
  AS_HD void move_and_log(int id, int dst, double now, int trigger) {
    int src = pool_of(id);
    int pos = pos_of(id);
    w.sync();
    for (int y = lane; y < MAX_INST; y += WD)
      if (y < sc().n_instances && y != id && sm->pool_of[y] == src && sm->pos_of[y] > pos) sm->pos_of[y]--;
    w.sync();
    lane0([&] {
      Uniform& U = u();
      sm->pool_of[id] = (int16_t)dst;
      sm->pos_of[id] = (int16_t)U.pool_n[dst];
      U.pool_n[src]--;
      U.pool_n[dst]++;
      U.n_flips++;
      log_decision(now, ARROW_DEC_FLIP, -1, id, trigger | (src << 3) | (dst << 5));
    });
#pragma unroll
    for (int k = 0; k < IPL; k++)
      if (st[k].id == id) st[k].pool = dst;
  }

  // ---------------------------------------------------- scheduler ------

  AS_HD void compute_delays(double now) {
    PROF_CLOCK(pd0);
#pragma unroll
    for (int k = 0; k < IPL; k++)
      if (st[k].id >= 0) delay_interval(st[k], now);
    dnow = now;
#ifdef ARROW_PROF
    w.sync();
#endif
    PROF_MARK(14, pd0);
  }

  // _argmin over one pool (insertion order), key = delay
  AS_HD int argmin_delay_pool(int pool) {
    return argmin_delay([&](const Inst& I) { return I.pool == pool; },
                        [&](const Inst& I) { return (uint32_t)pos_of(I.id); });
  }

  // Exact argmin of the predicted delay over the instances `sel` accepts,
  // first minimum by `tie` (scheduler.py:89-99), from the delay intervals of
  // compute_delays: only candidates whose interval reaches below every
  // candidate's upper end can be the minimum; when more than one can, they
  // fold exactly.
  template <class Sel, class Tie>
  AS_HD int argmin_delay(Sel sel, Tie tie_of) {
    uint64_t mk = ~0ull;
    bool cand[IPL];
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      cand[k] = st[k].id >= 0 && sel(st[k]);
      if (cand[k]) {
        const uint64_t x = okey(st[k].dhi);
        if (x < mk) mk = x;
      }
    }
    const uint32_t mhi = w.min_u32((uint32_t)(mk >> 32));
    const uint32_t mlo = w.min_u32((uint32_t)(mk >> 32) == mhi ? (uint32_t)mk : ~0u);
    mk = ((uint64_t)mhi << 32) | mlo;
    int ncont = 0, single = -1;
    bool cont[IPL];
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      cont[k] = cand[k] && okey(st[k].dlo) <= mk;
      const uint32_t m = w.ballot(cont[k]);
      ncont += popc32(m);
      if (m) single = ffs32(m) + WD * k;  // instance i lives on lane i % WD, slot i / WD
    }
    if (ncont == 0) return -1;
    if (ncont == 1) return single;  // the only candidate whose interval reaches the minimum
    {
#pragma unroll
      for (int k = 0; k < IPL; k++)
        if (cont[k]) delay_exact(st[k], dnow);
    }
    return argmin_inst([&](Inst& I, uint64_t& key, uint32_t& tie) {
      bool c = false;
#pragma unroll
      for (int k = 0; k < IPL; k++)
        if (&I == &st[k]) c = cont[k];
      if (!c) return false;
      key = okey(I.dly);
      tie = tie_of(I);
      return true;
    });
  }

  // fl(delay + own) <= thr for instance id (monotone in the delay, so both
  // interval ends on the same side decide it; otherwise fold exactly).
  AS_HD bool delay_within(int id, double own, double thr) {
    owner(id, [&](Inst& I) {
      int r;
      if (!I.dexact && I.dhi + own <= thr)
        r = 1;
      else if (!I.dexact && !(I.dlo + own <= thr))
        r = 0;
      else {
        delay_exact(I, dnow);
        r = I.dly + own <= thr ? 1 : 0;
      }
      u().tmp_i[0] = r;
    });
    const bool ok = u().tmp_i[0] != 0;
    w.sync();
    return ok;
  }

  AS_HD int argmin_tokens_pool(int pool) {
    return argmin_inst([&](Inst& I, uint64_t& key, uint32_t& tie) {
      if (I.pool != pool) return false;
      key = (uint64_t)(uint32_t)I.rtok;
      tie = (uint32_t)pos_of(I.id);
      return true;
    });
  }

  // members(DECODE) + members(P_TO_D) order
  AS_HD uint32_t decode_role_tie(int id) const {
    return (pool_of(id) == P_DECODE ? 0u : 256u) + (uint32_t)pos_of(id);
  }

  AS_HD bool decode_role(int id) const { return pool_of(id) == P_DECODE || pool_of(id) == P_P2D; }

  // _pool_mean_interval (scheduler.py:124-134): ordered Neumaier sum of the
  // non-None intervals of DECODE then P_TO_D members, divided by the count.
  AS_HD bool pool_mean_interval(double now, double* out) {
    const int nD = u().pool_n[P_DECODE];
    const int m = nD + u().pool_n[P_P2D];
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      Inst& I = st[k];
      if (I.id < 0 || !decode_role(I.id)) continue;
      int cpos = pool_of(I.id) == P_DECODE ? pos_of(I.id) : nD + pos_of(I.id);
      double v = 0.0;
      bool ok = interval(I, now, &v);
      sm->vals[cpos] = v;
      sm->valid[cpos] = ok ? 1 : 0;
    }
    w.sync();
    const MeanOut r = pool_mean_sum(sm->vals, sm->valid, m);
    w.sync();
    *out = r.v;
    return r.ok != 0;
  }

  // decode_load_is_low, scheduler.py:136-147
  AS_HD bool decode_load_is_low(double now) {
#ifdef ARROW_PROF
    PROF_CLOCK(pl0);
    const bool r = decode_load_is_low_(now);
    PROF_MARK(15, pl0);
    return r;
  }
  AS_HD bool decode_load_is_low_(double now) {
#endif
    bool mine = false;
    uint32_t mn = ~0u;
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      if (st[k].id >= 0 && decode_role(st[k].id)) {
        mine = true;
        if ((uint32_t)st[k].rtok < mn) mn = (uint32_t)st[k].rtok;
      }
    }
    if (w.ballot(mine) == 0) return false;
    uint32_t min_tokens = w.min_u32(mn);
    if ((double)min_tokens > sc().theta_d * (double)sc().max_tokens) return false;
    double mean;
    if (!pool_mean_interval(now, &mean)) return true;
    return mean <= sc().tpot_thr;
  }

  // try_move_decode_to_prefill, scheduler.py:258-276
  AS_HD int try_move_d2p(double now, int trigger) {
    if (!sc().enable_flips) return -1;
    if (u().pool_n[P_DECODE] + u().pool_n[P_P2D] <= 1) return -1;
    int cand = u().pool_n[P_P2D] > 0 ? P_P2D : P_DECODE;
    int chosen = argmin_tokens_pool(cand);
    int hdw = bcast_i(chosen, [&](Inst& I) { return has_decode_work(I) ? 1 : 0; });
    int dst = cand == P_DECODE ? (hdw ? P_D2P : P_PREFILL) : P_PREFILL;
    move_and_log(chosen, dst, now, trigger);
    return chosen;
  }

  // try_move_prefill_to_decode, scheduler.py:278-296 (delays must be current)
  AS_HD int try_move_p2d(double now, int trigger) {
    if (!sc().enable_flips) return -1;
    if (u().pool_n[P_PREFILL] + u().pool_n[P_D2P] <= 1) return -1;
    int cand = u().pool_n[P_D2P] > 0 ? P_D2P : P_PREFILL;
    int chosen = argmin_delay_pool(cand);
    int hpw = bcast_i(chosen, [&](Inst& I) { return has_prefill_work(I) ? 1 : 0; });
    int dst = cand == P_PREFILL ? (hpw ? P_P2D : P_DECODE) : P_DECODE;
    move_and_log(chosen, dst, now, trigger);
    return chosen;
  }

  AS_HD int rr_pick(int pool, int64_t counter) {
    int n = u().pool_n[pool];
    int want = (int)(counter % n);
    int id = -1;
#pragma unroll
    for (int k = 0; k < IPL; k++)
      if (st[k].id >= 0 && pool_of(st[k].id) == pool && pos_of(st[k].id) == want) id = st[k].id;
    uint32_t b = w.ballot(id >= 0);
    return w.shfl(id, ffs32(b));
  }

  // schedule_prefill / schedule_decode log one dispatch at a single code site
  // each; the choose_* bodies return (target | branch << 16), or -1.  The
  // t1 / t2 candidate tests run in one non-unrolled loop (one inlined copy of
  // the argmin and of the admission test instead of one per pool).
  static AS_HD int pack_choice(int t, int branch) { return (t & 0xffff) | (branch << 16); }   // >= 0
  static AS_HD int choice_target(int c) { return (int)(int16_t)(c & 0xffff); }

  // schedule_prefill, scheduler.py:151-195
  AS_HD int schedule_prefill(int rid, double now, double own) {
    const int c = choose_prefill(now, own);
    if (c < 0) return -1;                // no instance (status set)
    log_dispatch(now, ARROW_DEC_PREFILL_DISPATCH, rid, choice_target(c), c >> 16);
    return choice_target(c);
  }

  AS_HD int choose_prefill(double now, double own) {
    const int strat = sc().strategy;
    if (strat == ARROW_STRATEGY_ROUND_ROBIN) {
      int chosen = rr_pick(P_PREFILL, u().rr_p);
      w.sync();
      lane0([&] { u().rr_p++; });
      return pack_choice(chosen, ARROW_BR_ROUND_ROBIN);
    }
    compute_delays(now);
    if (strat == ARROW_STRATEGY_MINIMAL_LOAD) return pack_choice(argmin_delay_pool(P_PREFILL), ARROW_BR_MIN_LOAD);
    const double thr = sc().ttft_thr;
    int t1 = -1, t2 = -1;
#pragma unroll 1
    for (int c = 0; c < 2; c++) {       // t1 over PREFILL, then t2 over D_TO_P (scheduler.py:168-175)
      const int t = argmin_delay_pool(c == 0 ? P_PREFILL : P_D2P);
      if (c == 0) t1 = t; else t2 = t;
      if (t >= 0 && delay_within(t, own, thr)) return pack_choice(t, c == 0 ? ARROW_BR_ALG1_T1 : ARROW_BR_ALG1_T2);
    }
    if (sc().enable_flips && decode_load_is_low(now)) {
      int t3 = try_move_d2p(now, ARROW_TRIG_ALG1);
      if (t3 >= 0) return pack_choice(t3, ARROW_BR_ALG1_FLIP);
    }
    if (t1 >= 0) return pack_choice(t1, ARROW_BR_ALG1_FALLBACK);
    if (t2 >= 0) return pack_choice(t2, ARROW_BR_ALG1_FALLBACK);
    int chosen = argmin_delay([&](const Inst& I) { return decode_role(I.id); },
                              [&](const Inst& I) { return (uint32_t)decode_role_tie(I.id); });
    if (chosen < 0) {
      lane0([&] { set_status(ARROW_NO_INSTANCE); });
      return -1;
    }
    return pack_choice(chosen, ARROW_BR_ALG1_DEGENERATE);
  }

  // _decode_admissible, scheduler.py:214-218
  AS_HD bool decode_admissible(int id, int tokens, double now) {
    if ((int64_t)tokens > sc().max_tokens) return false;
    int r = 0;
    owner(id, [&](Inst& I) {
      double v;
      r = interval(I, now, &v) ? (v <= sc().tpot_thr ? 1 : 0) : 1;
      u().tmp_i[0] = r;
    });
    const bool ok = u().tmp_i[0] != 0;
    w.sync();
    return ok;
  }

  // schedule_decode, scheduler.py:199-254
  AS_HD int schedule_decode(int rid, int src, double now) {
    const int c = choose_decode(src, now);
    log_dispatch(now, ARROW_DEC_DECODE_DISPATCH, rid, choice_target(c), c >> 16);
    return choice_target(c);
  }

  AS_HD int choose_decode(int src, double now) {
    const int strat = sc().strategy;
    if (strat == ARROW_STRATEGY_ROUND_ROBIN) {
      int chosen = rr_pick(P_DECODE, u().rr_d);
      w.sync();
      lane0([&] { u().rr_d++; });
      return pack_choice(chosen, ARROW_BR_ROUND_ROBIN);
    }
    if (strat == ARROW_STRATEGY_MINIMAL_LOAD) return pack_choice(argmin_tokens_pool(P_DECODE), ARROW_BR_MIN_LOAD);
    if (decode_role(src)) return pack_choice(src, ARROW_BR_ALG2_ZERO_TRANSFER);
    int t1 = -1, t2 = -1, tok1 = 0, tok2 = 0;
#pragma unroll 1
    for (int c = 0; c < 2; c++) {       // t1 over DECODE, then t2 over P_TO_D (scheduler.py:225-234)
      const int t = argmin_tokens_pool(c == 0 ? P_DECODE : P_P2D);
      const int tok = t >= 0 ? bcast_i(t, [](Inst& I) { return I.rtok; }) : 0;
      if (c == 0) {
        t1 = t;
        tok1 = tok;
      } else {
        t2 = t;
        tok2 = tok;
      }
      if (t >= 0 && decode_admissible(t, tok, now)) return pack_choice(t, c == 0 ? ARROW_BR_ALG2_T1 : ARROW_BR_ALG2_T2);
    }
    if (sc().enable_flips) {
      compute_delays(now);
      int t3 = try_move_p2d(now, ARROW_TRIG_ALG2);
      if (t3 >= 0) return pack_choice(t3, ARROW_BR_ALG2_FLIP);
    }
    if (t1 >= 0 && (t2 < 0 || tok1 <= tok2)) return pack_choice(t1, ARROW_BR_ALG2_FALLBACK);
    if (t2 >= 0) return pack_choice(t2, ARROW_BR_ALG2_FALLBACK);
    return pack_choice(src, ARROW_BR_ALG2_FORCED_LOCAL);
  }

  // ------------------------------------------------------- handlers ----

  // returns the instance to kick (serial_tail), -1 if none
  AS_HD int on_arrival(double now) {
    const int rid = u().a;
    const double own = quad(sc().pred_a2, sc().pred_a1, sc().pred_a0, inl[rid]);
    w.sync();
    lane0([&] {
      Uniform& U = u();
      U.a = rid + 1;
      U.next_arrival = U.a < sc().n_requests ? arr[U.a] * sc().arrival_scale : 0.0;
    });
    PROF_CLOCK(ps0);
    int target = schedule_prefill(rid, now, own);
    PROF_MARK(16, ps0);
    if (target < 0) return -1;
    owner(target, [&](Inst& I) {
      if (I.wp_c >= L.qcap) {
        set_status(ARROW_BUFFER_OVERFLOW, ARROW_OVF_QUEUE);
        return;
      }
      int slot = ring(I.wp_h, I.wp_c, L.qcap);
      wp_rid(I.id)[slot] = rid;
      wp_term(I.id)[slot] = own;
      I.wp_c++;
      dd_add(I.ws_hi, I.ws_lo, own);
      if (fabs(own) > I.ws_max) I.ws_max = fabs(own);
    });
    return target;
  }

  // returns the decode target; *mig: a migration may start on it (serial_tail)
  AS_HD int on_prefill_complete(double now, bool* mig) {
    int rid = 0, src = 0;
    {
      Uniform& U = u();
      rid = p.fifo_rid[U.fifo_head];
      src = p.fifo_src[U.fifo_head];
    }
    w.sync();
    lane0([&] {
      Uniform& U = u();
      U.fifo_head = U.fifo_head + 1 == L.n_max ? 0 : U.fifo_head + 1;
      U.fifo_count--;
    });
    PROF_CLOCK(ps1);
    int target = schedule_decode(rid, src, now);
    PROF_MARK(17, ps1);
    const int in = inl[rid], g = outl[rid] - 1;
    owner(target, [&](Inst& I) {
      if (target == src) {
        I.parked--;           // adopt_local_decode: parked KV becomes the decode's
      } else {
        p.src[rid] = src;
        if (I.mq_c >= L.qcap) {
          set_status(ARROW_BUFFER_OVERFLOW, ARROW_OVF_QUEUE);
          return;
        }
        mq_rid(I.id)[ring(I.mq_h, I.mq_c, L.qcap)] = rid;
        if (I.mq_c == 0) I.mq_need = inl[rid] + (outl[rid] - 1);
        I.mq_c++;
        return;
      }
      if (I.wd_c >= L.qcap) {
        set_status(ARROW_BUFFER_OVERFLOW, ARROW_OVF_QUEUE);
        return;
      }
      wd_rid(I.id)[ring(I.wd_h, I.wd_c, L.qcap)] = rid;
      I.wd_c++;
      I.wgrowth += g;
      I.rtok += in;
    });
    *mig = target != src;
    return target;
  }

  AS_HD int on_migration_complete(int id, double now) {
    owner(id, [&](Inst& I) {
      int rid = I.mig_rid;
      I.mig_active = 0;
      I.kv_reserved -= inl[rid];
      I.kv_used += inl[rid];
      if (I.wd_c >= L.qcap) {
        set_status(ARROW_BUFFER_OVERFLOW, ARROW_OVF_QUEUE);
        return;
      }
      wd_rid(I.id)[ring(I.wd_h, I.wd_c, L.qcap)] = rid;
      I.wd_c++;
      I.wgrowth += outl[rid] - 1;
      I.rtok += inl[rid];
      u().tmp_i[1] = rid;
      u().tmp_i[2] = p.src[rid];
    });
    const int rid = u().tmp_i[1];
    const int src = u().tmp_i[2];
    w.sync();
    owner(src, [&](Inst& S) {
      S.kv_used -= inl[rid];   // release_parked
      S.parked--;
    });
    return src;                // serial_tail: migrations (id, src), then kicks (id, src)
  }

  // The serial handlers' trailing _start_migrations / _kick calls in program
  // order (engine.py:211-223, 228-236, 240-248), from one code site: each
  // inlined copy of kick() is ~300 instructions, and the occupancy build's
  // hot loop does not fit the instruction cache as it is.
  // The serial handlers' trailing _start_migrations (in program order, each
  // push sequenced at once); their _kick calls run in the shared kick phase.
  AS_HD void serial_migs(int m0, int m1, double now) {
    if (u().status != ARROW_OK) return;
#pragma unroll 1
    for (int q = 0; q < 2; q++) {
      const int id = q == 0 ? m0 : m1;
      if (id < 0) continue;
      owner(id, [&](Inst& I) {
        if (start_mig(I, now)) I.mig_seq = next_seq();
      });
    }
  }

  // The one inlined copy of kick(): every lane with want[k] starts its
  // instance's next iteration at tnow[k] (engine.py:170-177).
  AS_HD void kick_phase(const bool want[IPL], const double tnow[IPL], bool pushed[IPL]) {
#pragma unroll
    for (int k = 0; k < IPL; k++) pushed[k] = want[k] && kick(st[k], tnow[k]);
  }

  // Serial kicks sequenced in program order (k0 before k1).
  AS_HD void serial_kick_seqs(int k0, int k1, const bool pushed[IPL]) {
#pragma unroll 1
    for (int q = 0; q < 2; q++) {
      const int id = q == 0 ? k0 : k1;
      if (id < 0) continue;
      if (lane == lane_of(id)) {
#pragma unroll
        for (int k = 0; k < IPL; k++)
          if (st[k].id == id && pushed[k]) st[k].iter_seq = next_seq();
      }
      w.sync();
    }
  }

  AS_HD void write_snapshots(double now) {
    if (!(B->snapshots && HAVE_OM && om.snapshot_offset >= 0)) return;
    const int N = sc().n_instances;
    const int64_t base = u().n_snap;
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      Inst& I = st[k];
      if (I.id < 0) continue;
      int64_t slot = base + I.id;
      if (slot >= om.snapshot_capacity) continue;
      arrow_snapshot_t* s = B->snapshots + om.snapshot_offset + slot;
      double iv = 0.0;
      bool ok = interval(I, now, &iv);
      s->time = now;
      s->pred_delay = delay(I, now);
      s->avg_interval = ok ? iv : NAN;
      s->instance = I.id;
      s->pool = pool_of(I.id);
      s->running_tokens = I.rtok;
      s->kv_used = I.kv_used;
      s->queue_len = I.wp_c - I.pb_k;
      s->prefill_count = (I.rp_rid >= 0 ? 1 : 0) + I.wp_c;
      s->decode_count = I.R + I.wd_c + I.mq_c + (I.mig_active ? 1 : 0);
      s->reserved = 0;
    }
    w.sync();
    lane0([&] {
      if (base + N > om.snapshot_capacity && u().overflow == ARROW_OVF_NONE) u().overflow = ARROW_OVF_SNAPSHOTS;
      u().n_snap = base + N;
    });
  }

  // scheduler.monitor_tick, scheduler.py:300-335.  Returns true when the
  // tick changed nothing and the decode pool reported no interval (the
  // fixed point the stall fast path relies on).
  AS_HD bool monitor_tick(double now) {
    const arrow_scenario_t& s = sc();
    if (s.strategy != ARROW_STRATEGY_SLO_AWARE || !s.enable_flips) return true;
    const int flips0 = u().n_flips;
    double mean = 0.0;
    bool have = pool_mean_interval(now, &mean);
    if (have && mean > s.tpot_thr) {
      lane0([&] { u().breach += s.monitor_period; });
      if (u().breach >= s.breach_duration) {
        compute_delays(now);
        try_move_p2d(now, ARROW_TRIG_MONITOR_TPOT);
      }
    } else {
      lane0([&] { u().breach = 0.0; });
    }
    // aggregate decode load over DECODE + P_TO_D
    uint64_t agg = 0;
    bool mine = false;
#pragma unroll
    for (int k = 0; k < IPL; k++)
      if (st[k].id >= 0 && decode_role(st[k].id)) {
        agg += (uint64_t)(uint32_t)st[k].rtok;
        mine = true;
      }
    uint32_t members = w.ballot(mine);
    if (members == 0) return !have && u().n_flips == flips0;
    for (int off = WD / 2; off > 0; off >>= 1) agg += w.shfl(agg, (lane + off) & (WD - 1));
    agg = w.shfl(agg, 0);
    int m = 0;
    {
      int c = 0;
#pragma unroll
      for (int k = 0; k < IPL; k++) c += (st[k].id >= 0 && decode_role(st[k].id)) ? 1 : 0;
      m = (int)w.add_u32((uint32_t)c);
    }
    int64_t capacity = s.max_tokens * (int64_t)m;
    if (capacity == 0) {
      lane0([&] { set_status(ARROW_ZERO_DIVISION); });
      return false;
    }
    if ((double)agg / (double)capacity <= s.theta_busy) return !have && u().n_flips == flips0;
    // snapshot of PREFILL members in insertion order
    const int np = u().pool_n[P_PREFILL];
#pragma unroll
    for (int k = 0; k < IPL; k++)
      if (st[k].id >= 0 && pool_of(st[k].id) == P_PREFILL) sm->list[pos_of(st[k].id)] = st[k].id;
    w.sync();
    for (int j = 0; j < np; j++) {
      if (u().pool_n[P_PREFILL] + u().pool_n[P_D2P] <= 1) break;
      int x = sm->list[j];
      int busy_or_work = bcast_i(x, [&](Inst& I) { return (has_prefill_work(I) || I.busy) ? 1 : 0; });
      if (busy_or_work) continue;
      move_and_log(x, P_DECODE, now, ARROW_TRIG_MONITOR_IDLE);
    }
    w.sync();
    return !have && u().n_flips == flips0;
  }

  // ----------------------------------------------------- event loop ----

  AS_HD void init_scenario(int s) {
    sid = s;
    have_om = !LEAN && B->outmap != 0;
    if (HAVE_OM) om = B->outmap[s];
    lane0([&] {
      sm->sc = B->scenarios[s];
      Uniform& U = u();
      memset(&U, 0, sizeof(U));
      U.status = ARROW_OK;
      U.hash = 14695981039346656037ull;
      U.stall_time = NAN;
      const arrow_scenario_t& c = sm->sc;
      for (int i = 0; i < c.n_instances; i++) {
        int k = i < c.n_prefill_init ? P_PREFILL : P_DECODE;
        sm->pool_of[i] = (int16_t)k;
        sm->pos_of[i] = (int16_t)U.pool_n[k];
        U.pool_n[k]++;
      }
      U.seq = (uint32_t)c.n_requests;
      if (c.n_requests > 0) {
        U.tick_active = 1;
        U.tick_time = c.monitor_period;
        U.tick_seq = U.seq++;
      }
      U.a = 0;
      U.next_arrival = c.n_requests > 0 ? B->arrival[c.trace_offset] * c.arrival_scale : 0.0;
    });
    const arrow_scenario_t& c = sc();
    arr = B->arrival + c.trace_offset;
    inl = B->input_len + c.trace_offset;
    outl = B->output_len + c.trace_offset;
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      Inst& I = st[k];
      memset(&I, 0, sizeof(I));
      int id = lane + k * WD;
      I.id = id < c.n_instances ? id : -1;
      I.rp_rid = -1;
      I.min_f = 0x7fffffff;
      I.mig_rid = -1;
      I.pool = I.id >= 0 ? pool_of(I.id) : -1;
    }
    // Per-request state starts as "no token yet" only where it can be
    // observed: per-request outputs of a run that stops early.  A completed
    // run writes every first / last time before summarize() reads them.
    if (HAVE_OM && om.req_offset >= 0) {
      int32_t* rpf = B->req_prefill;
      int32_t* rdc = B->req_decode;
      int32_t* rdi = B->req_decode_iter;
      for (int r = lane; r < c.n_requests; r += WD) {
        p.first[r] = NAN;
        p.last[r] = NAN;
        if (rpf) rpf[om.req_offset + r] = -1;
        if (rdc) rdc[om.req_offset + r] = -1;
        if (rdi) rdi[om.req_offset + r] = -1;
      }
    }
    w.sync();
  }

  // Event selection (engine.py:267: pop the lexicographic (time, kind, seq)
  // minimum).  Pending events are split into
  //   * serial events: arrivals, PREFILL_COMPLETE, monitor ticks, migration
  //     completions, and "loud" iteration completions (those that push a
  //     PREFILL_COMPLETE, may start a migration, may drain a transition-pool
  //     instance, or emit nothing);
  //   * quiet iteration completions, whose handler touches only their own
  //     instance.
  // Let H be the earliest serial event.  Every quiet event before H whose
  // time is <= T = min_i(t_i + dl_i) over those quiet events (dl_i a lower
  // bound on the duration of the iteration instance i will start next) can be
  // executed in one round, lane-parallel: all of them precede every event the
  // round creates and every serial event, so the global order is preserved;
  // the round's pushes get their exact global sequence numbers by ranking the
  // round's events by (time, seq).  Returns:

  // Exact test of whether this completion has effects beyond its own
  // instance (engine.py:205-223): a PREFILL_COMPLETE push, a migration start
  // or a drained-pool move; or emits no token (stall counter).
  //  * migration: advance_migrations' gate (instance.py:140) compares
  //    X = kv_free - waiting growth with the queue head's need; executing
  //    the iteration raises X exactly by the KV of the decodes finishing at
  //    it and of released single-token prompts, and between handlers X
  //    never rises without a start_mig attempt, so the gate passes iff
  //    X_now + freed >= need.
  //  * drain (engine.py:183-192): the prefill / decode work left after the
  //    iteration is known from the pending batch.
  AS_HD bool quiet(const Inst& I) const {
    if (!I.busy || !I.pb_emit || I.pb_pc) return false;
    const int cur = I.it - 1;
    const int fin = I.min_f == cur ? I.min_f_cnt : 0;
    if (I.mq_c > 0 && !I.mig_active && (fin > 0 || I.pb_rel > 0)) {
      const int x = sc().kv_capacity - I.kv_used - I.kv_reserved - I.committed - I.wgrowth;
      const int freed = (fin > 0 ? I.held_min : 0) + I.pb_rel;
      if (x + freed >= I.mq_need) return false;
    }
    const int pk = I.pool;
    if (pk == P_P2D)
      return I.wp_c > I.pb_k || I.pb_rp_left || (I.pb_k > 0 && !I.pb_last_comp);
    if (pk == P_D2P) return I.mig_active || I.mq_c > 0 || I.wd_c > 0 || I.R - fin > 0;
    return true;
  }

  // Lower bound on the duration of the iteration this instance starts when
  // its pending iteration completes: its surviving running decodes are all
  // in the next batch (token-linear cost), otherwise the scenario minimum.
  AS_HD double next_duration_bound(const Inst& I) const {
    const int cur = I.it - 1;
    const int r_next = I.R - (I.min_f == cur ? I.min_f_cnt : 0);
    if (r_next >= 1) return sc().b1 * (double)r_next + sc().b0;
    return sc().min_iteration;
  }

  // The earliest serial event (time key, kind|seq, code); code -1 = none.
  struct Head {
    uint64_t k;
    uint32_t s;
    int code;
  };

  AS_HD void offer(Head& h, uint64_t k1, int kind, uint32_t seq, int c) const {
    const uint32_t k2 = ((uint32_t)kind << 28) | seq;
    if (h.code < 0 || k1 < h.k || (k1 == h.k && k2 < h.s)) {
      h.k = k1;
      h.s = k2;
      h.code = c;
    }
  }

  AS_HD void classify(Inst& I) const {
    I.ck = tkey(I.busy_until);
    I.cq = quiet(I) ? 1 : 0;
  }

  // Warp-uniform minimum of per-lane heads.
  AS_HD Head reduce_head(const Head& mine) {
    Head h;
    h.code = -1;
    h.k = ~0ull;
    h.s = ~0u;
    const int wl = warp_argmin(mine.k, mine.s, mine.code >= 0);
    if (wl >= 0) {
      h.k = w.shfl(mine.k, wl);
      h.s = w.shfl(mine.s, wl);
      h.code = w.shfl(mine.code, wl);
    }
    return h;
  }

  // Full rescan after a serial step: classify every pending iteration and
  // find the earliest serial event (lane 0 adds arrival, FIFO head, tick).
  AS_HD Head full_scan() {
    Head mine;
    mine.code = -1;
    mine.k = ~0ull;
    mine.s = ~0u;
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      Inst& I = st[k];
      if (I.id < 0) continue;
      if (I.busy) {
        classify(I);
        if (!I.cq) offer(mine, I.ck, EV_ITER, I.iter_seq, 2 * I.id + 1);
      }
      if (I.mig_active) offer(mine, tkey(I.mig_finish), EV_MIG, I.mig_seq, 2 * I.id);
    }
    if (lane == 0) {
      const Uniform& U = sm->u;
      if (U.a < sc().n_requests) offer(mine, tkey(U.next_arrival), EV_ARRIVAL, (uint32_t)U.a, 1000 + EV_ARRIVAL);
      if (U.fifo_count > 0)
        offer(mine, tkey(p.fifo_time[U.fifo_head]), EV_PREFILL, p.fifo_seq[U.fifo_head], 1000 + EV_PREFILL);
      if (U.tick_active) offer(mine, tkey(U.tick_time), EV_TICK, U.tick_seq, 1000 + EV_TICK);
    }
    return reduce_head(mine);
  }

  // Quiet iterations pending before the serial head.  None means the head
  // is the next event: no round and no burst (whose participants are quiet
  // iterations before the head) can run, so the serial step follows at once.
  AS_HD bool round_candidates(const Head& h, bool cand[IPL]) {
    bool any_cand = false;
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      const Inst& I = st[k];
      const uint32_t k2 = ((uint32_t)EV_ITER << 28) | I.iter_seq;
      cand[k] = I.id >= 0 && I.busy && I.cq && (h.code < 0 || I.ck < h.k || (I.ck == h.k && k2 < h.s));
      any_cand = any_cand || cand[k];
    }
    return w.any(any_cand);
  }

  // The candidates whose times are <= T = min(t_i + dl_i): one lane-parallel
  // round.
  AS_HD void round_select(const bool cand[IPL], bool part[IPL]) {
    uint64_t lim = ~0ull;
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      const Inst& I = st[k];
      if (cand[k]) {
        const uint64_t x = tkey(I.busy_until + next_duration_bound(I));
        if (x < lim) lim = x;
      }
    }
    const uint32_t hi = w.min_u32((uint32_t)(lim >> 32));
    const uint32_t lo = w.min_u32((uint32_t)(lim >> 32) == hi ? (uint32_t)lim : ~0u);
    const uint64_t cut = ((uint64_t)hi << 32) | lo;
#pragma unroll
    for (int k = 0; k < IPL; k++) part[k] = cand[k] && st[k].ck <= cut;
  }

  // One parallel round of quiet iteration completions; folds any loud
  // event the round created into the head.
  // Lane-parallel round, part 1: the participants' completions (their
  // kicks follow in the shared kick phase, then round_finish()).
  // serial: the loud ITERATION_COMPLETE of one instance (its owner lane is
  // the only participant): one inlined copy of iteration_complete() serves
  // both paths.
  AS_HD void round_complete(const bool part[IPL], uint64_t key1[IPL], uint32_t key2[IPL], double tnow[IPL],
                            int& completed, int& n_part, bool serial) {
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      key1[k] = 0;
      key2[k] = 0;
      tnow[k] = 0.0;
      if (!part[k]) continue;
      Inst& I = st[k];
      key1[k] = tkey(I.busy_until);
      key2[k] = I.iter_seq;
      tnow[k] = I.busy_until;
      n_part++;
      if (serial) {
        ATRACE("loud inst %d pc %d emit %d pool %d mq %d ma %d frees %d\n", I.id, I.pb_pc, I.pb_emit, pool_of(I.id),
               I.mq_c, I.mig_active, (int)(I.min_f == I.it - 1 || I.pb_rel));
#ifdef ARROW_PROF
        if (!I.pb_emit && !I.pb_pc) u().cyc_kind[25] += 1;   // token-less (silent) loud iterations
        if (I.pb_pc) u().cyc_kind[31] += 1;                  // PREFILL_COMPLETE-pushing ones
#endif
      }
      int done = 0;
      const int dst = iteration_complete(I, I.busy_until, done, serial);
      completed += done;
      if (serial) {
        u().n_iters++;
        u().tmp_i[0] = dst;
        u().completed += done;
      }
    }
    if (serial) w.sync();
  }

  AS_HD void round_finish(const bool part[IPL], const uint64_t key1[IPL], const uint32_t key2[IPL],
                          const bool pushed[IPL], int completed, int n_part, Head& h) {
    PROF_CLOCK(pr0);
    PROF_MARK(0, pr0);
    PROF_CLOCK(pr1);
    // exact push sequence: the round's pushes, in (time, seq) order of the
    // events that made them, continue the global counter
    const uint32_t base = u().seq;
    int pre[IPL];
#pragma unroll
    for (int k = 0; k < IPL; k++) pre[k] = 0;
    int my_push = 0;
#pragma unroll
    for (int kk = 0; kk < IPL; kk++) {
      uint32_t m = w.ballot(pushed[kk]);
      while (m) {
        const int j = ffs32(m);
        m &= m - 1;
        const uint64_t a = w.shfl(key1[kk], j);
        const uint32_t b = w.shfl(key2[kk], j);
#pragma unroll
        for (int k = 0; k < IPL; k++)
          if (pushed[k] && (a < key1[k] || (a == key1[k] && b < key2[k]))) pre[k]++;
      }
    }
    PROF_MARK(1, pr1);
    Head loud;
    loud.code = -1;
    loud.k = ~0ull;
    loud.s = ~0u;
#pragma unroll
    for (int k = 0; k < IPL; k++)
      if (pushed[k]) {
        Inst& I = st[k];
        I.iter_seq = base + (uint32_t)pre[k];
        my_push++;
        classify(I);
        if (!I.cq) offer(loud, I.ck, EV_ITER, I.iter_seq, 2 * I.id + 1);
      }
    if (w.any(loud.code >= 0)) {
      Head nl = reduce_head(loud);
      if (h.code < 0 || nl.k < h.k || (nl.k == h.k && nl.s < h.s)) h = nl;
    }
    // one reduction: pushes (<= 64) | participants (<= 64) << 7 | finished requests << 14
    const uint32_t packed = w.add_u32((uint32_t)my_push | ((uint32_t)n_part << 7) | ((uint32_t)completed << 14));
    const uint32_t total_push = packed & 127u;
    const uint32_t total_part = (packed >> 7) & 127u;
    const uint32_t total_done = packed >> 14;
    w.sync();
    lane0([&] {
      Uniform& U = u();
      seq_check(base + total_push);
      U.seq = base + total_push;
      U.esp = 0;  // every quiet event emits a token
      U.n_events += total_part;
      U.n_iters += total_part;
      U.n_rounds++;
      U.completed += (int)total_done;
    });
  }

  // ---------------------------------------------------- chain bursts ----
  //
  // An instance with no prefill work and no queued migration, in a non-
  // transition pool, can only run decode-only iterations until the next
  // serial event: every one of them emits tokens, pushes nothing but its
  // successor and touches nothing but its own state.  Such "chain-safe"
  // instances run their event chains in a local loop up to a horizon that
  // precedes every other pending event, then a merge of the per-instance
  // event lists (by time, ties by sequence) assigns the exact global push
  // sequence numbers the serial order would have produced.

  // A queued migration can only start when KV is freed, i.e. at the
  // completion of the iteration in which the earliest running decode
  // finishes (min_f); with no decode waiting, the chain runs fixed batches
  // of R decodes until then, so that completion time is exact arithmetic
  // and bounds the burst.
  // (Waiting decodes may be admitted without freed KV when they arrived
  // after the last kick, which would change R and min_f: such chains only
  // run when no migration can be pending.)
  AS_HD bool chain_safe(const Inst& I) const {
    const int pk = I.pool;
    return I.busy && I.cq && I.rp_rid < 0 && I.wp_c == 0 && (pk == P_PREFILL || pk == P_DECODE) &&
           !(I.mq_c > 0 && !I.mig_active && I.wd_c > 0);
  }

  // Lower bound on the completion time of the chain's first loud iteration
  // (the one where the earliest running decode finishes and the queued
  // migration's gate can open): busy_until + dur + ... + dur, `steps`
  // additions each rounded to nearest.  Every partial sum is <= T (the
  // closed form), so the accumulated rounding and the closed form's own are
  // below (steps + 4) ulp(T) <= (steps + 4) T 2^-52: L <= the exact sum.
  // Any lower bound keeps the burst exact (it only stops earlier); the
  // closed form replaces a serially dependent addition loop of up to
  // BURST_MAX steps per burst selection.
  AS_HD uint64_t chain_loud_bound(const Inst& I) const {
    if (I.mq_c == 0 || I.mig_active) return ~0ull;
    const int steps = I.min_f - (I.it - 1);   // >= 1: the pending event itself is quiet
    const double dur = sc().b1 * (double)I.R + sc().b0;
    const double T = I.busy_until + (double)steps * dur;
    const double L = T - (double)(steps + 4) * (T * 0x1p-52);
    return tkey(L > I.busy_until ? L : I.busy_until);
  }

  // Returns true and the horizon (events with key < hz are run) when some
  // chain-safe instance has an event before every other pending event;
  // `per` is the list segment each participant gets.
  // The horizon only has to be a lower bound of the exact one (a burst that
  // stops early is still exact: what it leaves runs in later steps), so the
  // warp minima it is built from use the high word of the order key alone --
  // one reduction each instead of a (high, low, sequence) argmin.
  AS_HD bool burst_select(const Head& h, Head& hz, bool safe[IPL], int& per) {
    uint32_t ns_hi = ~0u;  // high key word of the earliest non-safe pending iteration
    bool any_safe = false;
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      const Inst& I = st[k];
      safe[k] = I.id >= 0 && chain_safe(I);
      any_safe = any_safe || safe[k];
      if (I.id >= 0 && I.busy && !safe[k] && (uint32_t)(I.ck >> 32) < ns_hi) ns_hi = (uint32_t)(I.ck >> 32);
    }
    const bool some_safe = w.any(any_safe);
    ns_hi = w.min_u32(ns_hi);
#ifdef ARROW_PROF
    if (lane == 0) u().cyc_kind[21] += 1;                 // burst selections attempted
#endif
    if (!some_safe) return false;
    // limit = min(serial head, non-safe events rounded down to their high word)
    uint64_t lim_k = ~0ull;
    uint32_t lim_s = ~0u;
    bool lim = false;
    if (ns_hi != ~0u) {
      lim_k = (uint64_t)ns_hi << 32;
      lim_s = 0;
      lim = true;
    }
    if (h.code >= 0 && (!lim || h.k < lim_k)) {
      lim_k = h.k;
      lim_s = h.s;
      lim = true;
    }
    uint32_t t_hi = ~0u;
    int n_mine = 0;
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      const Inst& I = st[k];
      const uint32_t k2 = ((uint32_t)EV_ITER << 28) | I.iter_seq;
      safe[k] = safe[k] && (!lim || I.ck < lim_k || (I.ck == lim_k && k2 < lim_s));
      if (safe[k]) {
        n_mine++;
        if ((uint32_t)(I.ck >> 32) < t_hi) t_hi = (uint32_t)(I.ck >> 32);
      }
    }
    // both reductions issued back to back (independent), then the test
    const uint32_t n_part = w.add_u32((uint32_t)n_mine);
    t_hi = w.min_u32(t_hi);
#ifdef ARROW_PROF
    if (lane == 0) u().cyc_kind[22] += 1;                 // ... past the chain-safe test
#endif
    if (n_part == 0) return false;
    per = burst_share(n_part);
    // at most `per` events per instance: decode-only iterations last >= b1 + b0
    // (t0 <= the earliest participant's time)
    const double t0 = tkey_inv((uint64_t)t_hi << 32);
    uint64_t cap = tkey(t0 + (double)(per - 4) * (sc().b1 + sc().b0));
    {
      uint32_t l_hi = ~0u;
#pragma unroll
      for (int k = 0; k < IPL; k++)
        if (safe[k]) {
          const uint32_t bh = (uint32_t)(chain_loud_bound(st[k]) >> 32);
          if (bh < l_hi) l_hi = bh;
        }
      l_hi = w.min_u32(l_hi);
      const uint64_t lb = l_hi == ~0u ? ~0ull : ((uint64_t)l_hi << 32);
      if (lb < cap) cap = lb;
    }
    if (!lim || cap < lim_k) {
      hz.k = cap;
      hz.s = 0;
      hz.code = 0;
    } else {
      hz.k = lim_k;
      hz.s = lim_s;
      hz.code = 0;
    }
    bool run = false;
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      const uint32_t k2 = ((uint32_t)EV_ITER << 28) | st[k].iter_seq;
      safe[k] = safe[k] && (st[k].ck < hz.k || (st[k].ck == hz.k && k2 < hz.s));
      run = run || safe[k];
    }
    const bool go = w.any(run);
#ifdef ARROW_PROF
    if (lane == 0 && go) u().cyc_kind[23] += 1;           // ... that run a burst
#endif
    return go;
  }

  // Decode-only iteration chain of a chain-safe instance, from its pending
  // completion up to the horizon: exactly execute_iteration + _kick for
  // batches without prefill entries (instance.py:175-203, 229-288), with
  // the scenario constants held in registers.  Writes each event's time key
  // to `bk`; returns the events run and whether the last one pushed.
  AS_HD int chain_run(Inst& I, uint64_t hz_k, int limit, uint64_t* bk, int& completed, int& last_pushed) {
    const arrow_scenario_t& s = sc();
    const double b1 = s.b1, b0 = s.b0;
    const int kv_cap = s.kv_capacity;
    const int dcap = imin(s.max_batch, s.chunk_budget);
    double* ilog = (B->iterlog && HAVE_OM && om.iterlog_offset >= 0)
                       ? B->iterlog + om.iterlog_offset + (int64_t)I.id * om.iterlog_stride
                       : (double*)0;
    const int64_t ilog_cap = ilog ? om.iterlog_stride : 0;
    double* e = em(I.id);
    int c = 0;
    double t = I.busy_until;
    uint64_t key = I.ck;
    last_pushed = 0;
    for (;;) {
      const int cur = I.it - 1;
      // Steady stretch: no decode finishes before iteration min_f, no decode
      // is waiting, so every completion up to there applies the same batch
      // of R decodes and starts the next one (instance.py:187-191, 254-288):
      // only the emission, the event key and t += b1*R + b0 (the very
      // expression the general path evaluates) change per event; the
      // counters advance in bulk afterwards.
      if (!ilog && I.wd_c == 0 && I.min_f > cur && I.pb_ndec == I.R && I.R > 0 && I.R <= dcap) {
        const int R = I.R;
        const double dur = b1 * (double)R + b0;
        int room = (int)L.ecap - I.em_c;
        int kmax = I.min_f - cur;  // events cur, cur+1, ..., min_f - 1
        if (kmax > room) kmax = room;
        if (kmax > limit - c) kmax = limit - c;
        if (kmax >= 2) {
          int wpos = ring(I.em_h, I.em_c, L.ecap);
          const int ecap = (int)L.ecap;
          const double t_first = t;
          int k = 0;
          bool stop = false;
          double t_emit = t;
          while (k < kmax) {
            e[wpos] = t;             // the event at t: emission (cur + k)
            wpos = wpos + 1 == ecap ? 0 : wpos + 1;
            t_emit = t;
            bk[c++] = key;
            k++;
            t = t + dur;             // the iteration it starts
            key = tkey(t);
            if (key >= hz_k) {
              stop = true;
              break;
            }
          }
          I.kv_used += R * k;
          I.committed -= R * k;
          I.rtok += R * k;
          if (I.em_c == 0) I.em_first = t_first;
          I.em_c += k;
          I.em_last = t_emit;
          I.it += k;
          I.busy_until = t;
          I.ck = key;
          if (stop) {
            last_pushed = 1;
            return c;
          }
          if (c >= limit) {  // the horizon bounds the count; never taken
            set_status(ARROW_INTERNAL);
            return c;
          }
          continue;
        }
      }
      if (ilog) {
        if (cur < ilog_cap)
          ilog[cur] = t;
        else if (u().overflow == ARROW_OVF_NONE)
          u().overflow = ARROW_OVF_ITERLOG;
      }
      const int nd = I.pb_ndec;
      I.kv_used += nd;
      I.committed -= nd;
      I.rtok += nd;
      if (I.min_f == cur) {
        int* rr = run_rid(I.id);
        int* rf = run_f(I.id);
        int m = 0x7fffffff, mc = 0, mh = 0;
        int j = 0;
        while (j < I.R) {
          const int f = rf[j];
          if (f == cur) {
            const int rid = rr[j];
            const int held = inl[rid] + outl[rid] - 1;
            I.kv_used -= held;
            I.rtok -= held;
            p.last[rid] = t;
            completed++;
            I.R--;
            rr[j] = rr[I.R];
            rf[j] = rf[I.R];
          } else {
            const int hh = inl[rr[j]] + outl[rr[j]] - 1;
            if (f < m) {
              m = f;
              mc = 1;
              mh = hh;
            } else if (f == m) {
              mc++;
              mh += hh;
            }
            j++;
          }
        }
        I.min_f = m;
        I.min_f_cnt = mc;
        I.held_min = mh;
      }
      // emission ring (lazy pruning, see interval())
      if (I.em_c >= L.ecap) {
        emit(I, t);
      } else {
        e[ring(I.em_h, I.em_c, L.ecap)] = t;
        if (I.em_c == 0) I.em_first = t;
        I.em_last = t;
        I.em_c++;
      }
      bk[c] = key;
      c++;
      // _kick: running decodes, then waiting decodes FCFS under the growth gate
      int nd2 = I.R;
      if (I.wd_c > 0 && nd2 < dcap) {
        int kvf = kv_cap - I.kv_used - I.kv_reserved - I.committed;
        const int* wd = wd_rid(I.id);
        int ad = 0;
        while (ad < I.wd_c && nd2 < dcap) {
          const int g = outl[wd[ring(I.wd_h, ad, L.qcap)]] - 1;
          if (g > kvf) break;
          kvf -= g;
          nd2++;
          ad++;
        }
        if (ad > 0) {
          const int ncur = I.it;
          int* rr = run_rid(I.id);
          int* rf = run_f(I.id);
          int32_t* dit = (B->req_decode_iter && HAVE_OM && om.req_offset >= 0)
                             ? B->req_decode_iter + om.req_offset
                             : (int32_t*)0;
          for (int j = 0; j < ad; j++) {
            const int rid = wd[ring(I.wd_h, j, L.qcap)];
            const int g = outl[rid] - 1;
            const int f = ncur + g - 1;
            if (I.R >= L.rcap) {
              set_status(ARROW_BUFFER_OVERFLOW, ARROW_OVF_RUNNING);
              I.busy = 0;
              return c;
            }
            rr[I.R] = rid;
            rf[I.R] = f;
            I.R++;
            const int held = inl[rid] + g;
            if (f < I.min_f) {
              I.min_f = f;
              I.min_f_cnt = 1;
              I.held_min = held;
            } else if (f == I.min_f) {
              I.min_f_cnt++;
              I.held_min += held;
            }
            I.committed += g;
            I.wgrowth -= g;
            if (dit) dit[rid] = ncur;
          }
          I.wd_h = ring(I.wd_h, ad, L.qcap);
          I.wd_c -= ad;
        }
      } else if (I.R > dcap) {
        set_status(ARROW_INTERNAL);
      }
      if (nd2 == 0) {             // nothing startable: the chain ends
        I.busy = 0;
        I.pb_ndec = 0;
        return c;
      }
      I.it++;
      I.pb_ndec = nd2;
      t = t + (b1 * (double)nd2 + b0);
      key = tkey(t);
      I.busy_until = t;
      I.ck = key;
      last_pushed = 1;
      if (key >= hz_k) return c;
      if (c >= limit) {           // the horizon bounds the count; never taken
        set_status(ARROW_INTERNAL);
        return c;
      }
      last_pushed = 0;
    }
  }

  static AS_HD int lower_bound_u64(const uint64_t* a, int n, uint64_t x) {
    int lo = 0, hi = n;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (a[mid] < x)
        lo = mid + 1;
      else
        hi = mid;
    }
    return lo;
  }


  AS_HD void run_burst(const bool safe[IPL], const Head& hz, int per, Head& h) {
    // segments: participant rank (slot-major, then lane) x per
    int rank[IPL];
    int base_rank = 0;      // after the loop: the number of participants
    {
#pragma unroll
      for (int kk = 0; kk < IPL; kk++) {
        const uint32_t m = w.ballot(safe[kk]);
        rank[kk] = base_rank + popc32(m & ((1u << lane) - 1u));
        base_rank += popc32(m);
      }
    }
    PROF_CLOCK(pb0);
    int completed = 0, events = 0, pushes = 0;
    int lastp[IPL];
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      lastp[k] = 0;
      Inst& I = st[k];
      if (!safe[k]) {
        if (I.id >= 0) sm->bcount[I.id] = 0;
        continue;
      }
      const int off = rank[k] * per;
      sm->boff[I.id] = off;
      sm->bseq[I.id] = I.iter_seq;
      const int c = chain_run(I, hz.k, per, sm->blist + off, completed, lastp[k]);
      sm->bcount[I.id] = c;
      sm->blast[I.id] = lastp[k];
      events += c;
      pushes += c - 1 + lastp[k];
    }
    const uint32_t base = u().seq;
    if (lane == 0) sm->btie = 0;
    w.sync();
    PROF_MARK(12, pb0);
    PROF_CLOCK(pb1);
    // Sequence numbers only order events with equal times, and the pushes
    // inside a burst belong to events already executed: what the final
    // pending push of each chain must carry is its order relative to the
    // other chains' final pushes (by the time of the event that pushed it)
    // and a value in [base, base + total pushes), above every earlier push
    // and below every later one.  Rank among the finals gives exactly that;
    // equal final times fall back to the sequential merge below, which
    // reproduces the full (time, seq) order.
    int before[IPL];
    if (IPL == 1) {
      // Sharper still: the finals' relative order only matters among
      // finals whose pushed events have equal times.  When every pushed
      // event time is distinct (one match), lane order is as good as rank
      // order and the merge is two votes.
      const bool fin = safe[0] && lastp[0];
      const uint32_t fm = w.ballot(fin);
      // a 32-bit fold of the pushed time key (match.any on 32 bits is cheaper
      // than on 64): equal keys fold equal; distinct keys that happen to
      // collide only send the burst down the exact merge below
      const uint64_t nk = tkey(st[0].busy_until);
      const uint32_t hv = fin ? ((uint32_t)nk ^ ((uint32_t)(nk >> 32) * 0x9E3779B1u)) : 0u;
      const uint32_t peers = w.match_any_u32(hv) & fm;
      const bool dup = w.any(fin && (peers & (peers - 1u)) != 0);
      if (!dup) {
        const uint32_t packed = w.add_u32((uint32_t)events | ((uint32_t)completed << 16));
        // every chain pushes after each event but possibly its last:
        // pushes = events - participants + finals (no second reduction)
        const uint32_t total_push = (packed & 0xffffu) - (uint32_t)base_rank + (uint32_t)popc32(fm);
        if (fin) st[0].iter_seq = base + total_push - (uint32_t)popc32(fm) + (uint32_t)popc32(fm & ((1u << lane) - 1u));
        PROF_MARK(13, pb1);
        burst_finish(safe, base, packed, total_push, h);
        return;
      }
    }
    uint64_t xlast[IPL];  // key of each chain's final (pending-push) event
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      before[k] = 0;
      xlast[k] = ~0ull;
      if (st[k].id < 0) continue;
      const int id = st[k].id;
      if (safe[k] && lastp[k]) xlast[k] = sm->blist[sm->boff[id] + sm->bcount[id] - 1];
      sm->bfinal[id] = xlast[k];
    }
    const int n_final = (int)w.add_u32((uint32_t)(
        (IPL > 0 && safe[0] && lastp[0] ? 1 : 0) + (IPL > 1 && safe[IPL - 1] && lastp[IPL - 1] ? 1 : 0)));
    w.sync();
    bool tie_seen = false;
#pragma unroll
    for (int kk = 0; kk < IPL; kk++) {
      // only the other finals matter: walk the warp's final-push mask
      uint32_t m = w.ballot(safe[kk] && lastp[kk]);
      while (m) {
        const int j = ffs32(m);
        m &= m - 1;
        const int other = j + WD * kk;  // instance i lives on lane i % WD, slot i / WD
        const uint64_t v = sm->bfinal[other];
#pragma unroll
        for (int k = 0; k < IPL; k++) {
          if (!(safe[k] && lastp[k]) || st[k].id == other) continue;
          before[k] += (int)(v < xlast[k]);
          tie_seen = tie_seen || v == xlast[k];
        }
      }
    }
    if (tie_seen) sm->btie = 1;
    const uint32_t packed = w.add_u32((uint32_t)events | ((uint32_t)completed << 16));
    const uint32_t total_push = w.add_u32((uint32_t)pushes);
    w.sync();
    const int tie = sm->btie;
    if (!tie) {
#pragma unroll
      for (int k = 0; k < IPL; k++)
        if (safe[k] && lastp[k]) st[k].iter_seq = base + total_push - (uint32_t)n_final + (uint32_t)before[k];
    } else {
      // sequential merge of all chains in (time, seq) order; bseq[i] holds
      // the sequence of chain i's current head event
      lane0([&] {
        ATRACE("burst tie fallback base=%u\n", base);
        const int N = sc().n_instances;
        int* act = sm->list;
        int na = 0;
        for (int i = 0; i < N; i++) {
          if (sm->bcount[i] > 0) {
            act[na++] = i;
            sm->bhead[i] = 0;
          }
        }
        uint32_t seq = base;
        while (na > 0) {
          int best = 0;
          uint64_t bk0 = sm->blist[sm->boff[act[0]] + sm->bhead[act[0]]];
          for (int a2 = 1; a2 < na; a2++) {
            const int i = act[a2];
            const uint64_t kk = sm->blist[sm->boff[i] + sm->bhead[i]];
            // (mutant "tie": equal keys merged in reversed order)
            if (kk < bk0 || (kk == bk0 && (MUTANT("tie") ? sm->bseq[i] > sm->bseq[act[best]]
                                                          : sm->bseq[i] < sm->bseq[act[best]]))) {
              best = a2;
              bk0 = kk;
            }
          }
          const int i = act[best];
          const int hd = sm->bhead[i];
          const bool pushed = hd < sm->bcount[i] - 1 || sm->blast[i];
          if (pushed) sm->bseq[i] = seq++;
          sm->bhead[i] = hd + 1;
          if (hd + 1 >= sm->bcount[i]) act[best] = act[--na];
        }
      });
#pragma unroll
      for (int k = 0; k < IPL; k++)
        if (safe[k] && lastp[k]) st[k].iter_seq = sm->bseq[st[k].id];
    }
    PROF_MARK(13, pb1);
    burst_finish(safe, base, packed, total_push, h);
  }

  // a chain stopped at its migration bound leaves a loud pending event;
  // counters
  AS_HD void burst_finish(const bool safe[IPL], uint32_t base, uint32_t packed, uint32_t total_push, Head& h) {
    Head loud;
    loud.code = -1;
    loud.k = ~0ull;
    loud.s = ~0u;
#pragma unroll
    for (int k = 0; k < IPL; k++)
      if (safe[k] && st[k].busy) {
        classify(st[k]);
        if (!st[k].cq) offer(loud, st[k].ck, EV_ITER, st[k].iter_seq, 2 * st[k].id + 1);
      }
    if (w.any(loud.code >= 0)) {
      Head nl = reduce_head(loud);
      if (h.code < 0 || nl.k < h.k || (nl.k == h.k && nl.s < h.s)) h = nl;
    }
    lane0([&] {
      Uniform& U = u();
      seq_check(base + total_push);
      U.seq = base + total_push;
      U.esp = 0;
      U.n_events += packed & 0xffffu;
      U.n_iters += packed & 0xffffu;
      U.completed += (int)(packed >> 16);
      U.n_bursts++;
    });
  }

  AS_HD bool only_tick_pending() {
    bool active = false;
#pragma unroll
    for (int k = 0; k < IPL; k++) active = active || (st[k].id >= 0 && (st[k].busy || st[k].mig_active));
    if (w.any(active)) return false;
    const Uniform& U = sm->u;
    return U.a >= sc().n_requests && U.fifo_count == 0 && U.tick_active && U.completed < sc().n_requests;
  }



#ifdef ARROW_AUDIT
  // RunConfig.audit (engine.py:279-282): Instance.audit() (instance.py:364-
  // 378) and PoolSet.check_partition() (pools.py:127-137) after every step.
  // The incremental counters are recomputed from the queues themselves: KV
  // held by running decodes (prompt + generated), by the partial and the
  // pending prefill chunks, by waiting decodes and by prompts parked for a
  // PREFILL_COMPLETE or a migration (found in the FIFO and in every
  // instance's migration queue); KV reserved by the active migration; the
  // growth and running-token sums; pool membership.  A mismatch ends the run
  // with ARROW_AUDIT_FAILED (the shim raises AssertionError).
  AS_HD void audit_state() {
    const int N = sc().n_instances;
    lane0([&] {
      for (int i = 0; i < N; i++) sm->aud_parked_kv[i] = sm->aud_parked_n[i] = 0;
      const Uniform& U = u();
      for (int c = 0; c < U.fifo_count; c++) {
        const int slot = ring(U.fifo_head, c, L.n_max);
        sm->aud_parked_kv[p.fifo_src[slot]] += inl[p.fifo_rid[slot]];
        sm->aud_parked_n[p.fifo_src[slot]]++;
      }
    });
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      const Inst& I = st[k];
      if (I.id < 0) continue;
      for (int c = 0; c < I.mq_c + (I.mig_active ? 1 : 0); c++) {
        const int rid = c < I.mq_c ? mq_rid(I.id)[ring(I.mq_h, c, L.qcap)] : I.mig_rid;
        w.atomic_add_shared(&sm->aud_parked_kv[p.src[rid]], inl[rid]);
        w.atomic_add_shared(&sm->aud_parked_n[p.src[rid]], 1);
      }
    }
    w.sync();
    bool bad = false;
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      const Inst& I = st[k];
      if (I.id < 0) continue;
      const int lc = I.it - 1 - (I.busy ? 1 : 0);      // last completed iteration
      int64_t held = 0, committed = 0, rtok = 0, wgrowth = 0;
      for (int j = 0; j < I.R; j++) {                  // running decodes
        const int rid = run_rid(I.id)[j];
        const int f = run_f(I.id)[j];
        const int g = outl[rid] - 1;
        const int gen = g - (f - lc);
        bad = bad || gen < 0 || gen >= g;
        held += inl[rid] + gen;
        committed += f - lc;
        rtok += inl[rid] + gen;
      }
      for (int j = 0; j < I.wd_c; j++) {               // waiting decodes hold their prompt
        const int rid = wd_rid(I.id)[ring(I.wd_h, j, L.qcap)];
        held += inl[rid];
        wgrowth += outl[rid] - 1;
        rtok += inl[rid];
      }
      if (I.rp_rid >= 0) held += I.rp_done + (I.busy ? I.pb_rp_chunk : 0);
      if (I.busy)                                      // prompts admitted by the pending batch
        for (int j = 0; j < I.pb_k; j++) held += j < I.pb_k - 1 ? inl[wp_rid(I.id)[ring(I.wp_h, j, L.qcap)]] : I.pb_last_chunk;
      held += sm->aud_parked_kv[I.id];
      bad = bad || held != I.kv_used || committed != I.committed || rtok != I.rtok || wgrowth != I.wgrowth;
      bad = bad || sm->aud_parked_n[I.id] != I.parked;
      bad = bad || I.kv_reserved != (I.mig_active ? inl[I.mig_rid] : 0);
      bad = bad || I.kv_used < 0 || I.kv_reserved < 0 || I.kv_used + I.kv_reserved > sc().kv_capacity;
      bad = bad || I.pool != sm->pool_of[I.id] || I.pool < 0 || I.pool > 3;
    }
    if (lane == 0) {                                   // partition: counts and distinct positions per pool
      int cnt[4] = {0, 0, 0, 0};
      for (int i = 0; i < N; i++) {
        const int pk = sm->pool_of[i];
        if (pk < 0 || pk > 3) {
          bad = true;
          continue;
        }
        cnt[pk]++;
        for (int j = 0; j < i; j++) bad = bad || (sm->pool_of[j] == pk && sm->pos_of[j] == sm->pos_of[i]);
      }
      for (int q = 0; q < 4; q++) bad = bad || cnt[q] != u().pool_n[q];
    }
    if (w.any(bad)) lane0([&] { set_status(ARROW_AUDIT_FAILED); });
    w.sync();
  }
#define AUDIT_STEP() audit_state()
#else
#define AUDIT_STEP() \
  do {               \
  } while (0)
#endif

  AS_HD void simulate() {
    const int64_t limit = sc().stall_limit;
    Head h = full_scan();
    for (;;) {
      bool part[IPL];
      bool cand[IPL];
      Head hz;
      int per = 0;
      // shared kick phase inputs: a lane-parallel round's participants, or the
      // serial handler's kick targets (tk0 before tk1)
      bool round = false;
      bool want[IPL];
      double tnow[IPL];
      uint64_t key1[IPL];
      uint32_t key2[IPL];
      int completed = 0, n_part = 0;
      int tk0 = -1, tk1 = -1;
      int iter_id = -1, serial_tm0 = -1, serial_tm1 = -1;
      double now = 0.0;
#ifdef ARROW_PROF
      int prof_kind = 0;
#endif
      PROF_CLOCK(c0);
      if (round_candidates(h, cand)) {
        const bool bsel = burst_select(h, hz, part, per);
        PROF_MARK(8, c0);
        if (bsel) {
          PROF_CLOCK(cb);
          run_burst(part, hz, per, h);
          AUDIT_STEP();
          PROF_MARK(9, cb);
          PROF_ADD(cyc_burst, c0);
          const int status = u().status;
          w.sync();
          if (status != ARROW_OK) return;
          continue;
        }
        PROF_CLOCK(cr);
        round_select(cand, part);
        PROF_MARK(10, cr);
        round = true;
      } else {
      PROF_MARK(8, c0);
      if (h.code < 0) break;
      const int ev = h.code;
      now = tkey_inv(h.k);
      lane0([&] {
        seq_check(u().seq);
        u().now = now;
        u().esp++;
        u().n_events++;
        u().n_serial++;
        ATRACE("ev %d t=%.17g esp=%lld\n", ev, now, (long long)u().esp);
      });
#ifdef ARROW_PROF
      prof_kind = ev >= 1000 ? ev - 1000 : ((ev & 1) ? 5 : 6);
      if (lane == 0) u().cyc_kind[24 + prof_kind] += 1;   // event counts by kind
      PROF_MARK(20, c0);                                   // selection + bookkeeping up to here
#endif
      int tm0 = -1, tm1 = -1;   // serial_migs() arguments
      if (ev >= 1000) {
        int kind = ev - 1000;
        if (kind == EV_ARRIVAL) {
          tk0 = on_arrival(now);
        } else if (kind == EV_PREFILL) {
          bool mig = false;
          tk0 = on_prefill_complete(now, &mig);
          if (mig) tm0 = tk0;
        } else {
          lane0([&] { u().n_ticks++; });
          write_snapshots(now);
          bool fixed = monitor_tick(now);
          bool idle = only_tick_pending();
          bool healthy = u().status == ARROW_OK && u().esp <= limit;
          w.sync();
          lane0([&] {
            Uniform& U = u();
            if (U.completed < sc().n_requests) {
              U.tick_time = now + sc().monitor_period;
              U.tick_seq = next_seq();
            } else {
              U.tick_active = 0;
            }
          });
          if (fixed && idle && healthy) {
            // Nothing but ticks can ever happen again and each tick is a
            // no-op: count them down to the watchdog (engine.py:283-284).
            lane0([&] {
              Uniform& U = u();
              double t = now;
              while (U.esp <= limit) {
                t = U.tick_time;
                U.tick_time = t + sc().monitor_period;
                U.esp++;
                U.n_events++;
                U.n_ticks++;
              }
              U.now = t;
            });
            now = u().now;
          }
        }
      } else {
        int id = ev >> 1;
        if (ev & 1) {
          iter_id = id;               // the ITERATION_COMPLETE handler runs in round_complete() below
#pragma unroll
          for (int k = 0; k < IPL; k++) part[k] = st[k].id == id;
        } else {
          const int src = on_migration_complete(id, now);
          tm0 = tk0 = id;
          tm1 = tk1 = src;
        }
      }
      serial_tm0 = tm0;
      serial_tm1 = tm1;
      }   // serial step (handlers)
      if (round || iter_id >= 0) {
        PROF_CLOCK(pi0);
        round_complete(part, key1, key2, tnow, completed, n_part, !round);
        PROF_MARK(19, pi0);
      }
      if (round) {
#pragma unroll
        for (int k = 0; k < IPL; k++) want[k] = part[k];
      } else {
      int tm0 = serial_tm0, tm1 = serial_tm1;
      if (iter_id >= 0) {           // engine.py:219-223: drained move, then migrations and the kick
        const int dst = u().tmp_i[0];
        w.sync();
        if (dst >= 0) move_and_log(iter_id, dst, now, ARROW_TRIG_DRAINED);
        tm0 = tk0 = iter_id;
      }
      serial_migs(tm0, tm1, now);
      const bool ok = u().status == ARROW_OK;
#pragma unroll
      for (int k = 0; k < IPL; k++) {
        want[k] = ok && st[k].id >= 0 && (st[k].id == tk0 || st[k].id == tk1);
        tnow[k] = now;
      }
      }   // serial step
      bool pushed[IPL];
      PROF_CLOCK(pt0);
      kick_phase(want, tnow, pushed);       // the one inlined copy of kick()
      PROF_MARK(18, pt0);
      if (round) {
        PROF_CLOCK(cx);
        round_finish(part, key1, key2, pushed, completed, n_part, h);
        AUDIT_STEP();
        PROF_MARK(11, cx);
        PROF_ADD(cyc_round, c0);
        const int status = u().status;
        w.sync();
        if (status != ARROW_OK) return;
        continue;
      }
      serial_kick_seqs(tk0, tk1, pushed);
      AUDIT_STEP();
      const int status = u().status;
      const int64_t esp = u().esp;
      w.sync();
      if (status != ARROW_OK) return;
      if (esp > limit) {
        lane0([&] {
          u().status = ARROW_STALLED;
          u().stall_time = now;
        });
        return;
      }
      PROF_CLOCK(c1);
      h = full_scan();
      PROF_ADD(cyc_serial, c0);
#ifdef ARROW_PROF
      if (lane == 0) {
        u().cyc_kind[prof_kind] += c1 - c0;
        u().cyc_kind[7] += clock_now() - c1;
      }
#endif
    }
    // end-of-run checks, engine.py:286-290
    lane0([&] {
      if (u().seq >= SEQ_LIMIT) set_status(ARROW_BUFFER_OVERFLOW, ARROW_OVF_SEQ);
    });
    if (u().status != ARROW_OK) return;
    const int completed = u().completed;
    w.sync();
    if (completed != sc().n_requests) {
      lane0([&] { u().status = ARROW_INCOMPLETE; });
      return;
    }
    bool dirty = false;
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      const Inst& I = st[k];
      if (I.id < 0) continue;
      dirty = dirty || I.busy || I.R || I.rp_rid >= 0 || I.wp_c || I.wd_c || I.mq_c || I.mig_active ||
              I.parked || I.kv_used || I.kv_reserved;
    }
    if (w.any(dirty)) lane0([&] { u().status = ARROW_NOT_DRAINED; });
  }

  AS_HD void write_diag() {
    if (!(B->diag && HAVE_OM && om.diag_offset >= 0)) return;
#pragma unroll
    for (int k = 0; k < IPL; k++) {
      const Inst& I = st[k];
      if (I.id < 0) continue;
      arrow_instdiag_t* d = B->diag + om.diag_offset + I.id;
      d->busy_until = I.busy ? I.busy_until : NAN;
      d->pool = pool_of(I.id);
      d->kv_used = I.kv_used;
      d->running = I.R + (I.rp_rid >= 0 ? 1 : 0) + (I.busy ? I.pb_k : 0);
      d->waiting = (I.wp_c - (I.busy ? I.pb_k : 0)) + I.wd_c;
      d->migrating = I.mq_c;
      d->reserved = 0;
    }
    w.sync();
  }

  // Radix select of the k-th smallest (0-based) non-negative double.
  AS_HD double select_kth(const double* v, int n, int kth) {
    uint64_t prefix = 0, mask = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int b = lane; b < 256; b += WD) sm->hist[b] = 0;
      w.sync();
      for (int i = lane; i < n; i += WD) {
        uint64_t key = okey(v[i]);
        if ((key & mask) == prefix) w.atomic_add_shared(&sm->hist[(key >> shift) & 255], 1);
      }
      w.sync();
      lane0([&] {
        int acc = 0, b = 0;
        for (; b < 256; b++) {
          if (acc + sm->hist[b] > u().tmp_i[3]) break;
          acc += sm->hist[b];
        }
        u().tmp_i[3] -= acc;
        u().tmp_i[2] = b;
      });
      prefix |= (uint64_t)u().tmp_i[2] << shift;
      mask |= (uint64_t)255 << shift;
      w.sync();
    }
    return okey_inv(prefix);
  }

  // compute_metrics over the run's records (report.py:55-74, core.py:105-156)
  AS_HD void summarize(arrow_summary_t* out) {
    const arrow_scenario_t& c = sc();
    const int n = c.n_requests;
    uint32_t ok_cnt = 0;
    uint64_t kmax = 0, kmin = ~0ull;
    for (int r = lane; r < n; r += WD) {
      double a = arr[r] * c.arrival_scale;
      double f = p.first[r], l = p.last[r];
      int m = outl[r];
      double tt = f - a;
      double tp = m == 1 ? 0.0 : (l - f) / (double)(m - 1);
      p.ttft[r] = tt;
      p.tpot[r] = tp;
      ok_cnt += (tt <= c.ttft_slo && tp <= c.tpot_slo) ? 1u : 0u;
      uint64_t kl = okey(l), ka = okey(a);
      if (kl > kmax) kmax = kl;
      if (ka < kmin) kmin = ka;
    }
    uint32_t n_ok = w.add_u32(ok_cnt);
    // 64-bit max/min via two-step 32-bit redux
    uint32_t hi = w.max_u32((uint32_t)(kmax >> 32));
    uint32_t lo = w.max_u32((uint32_t)(kmax >> 32) == hi ? (uint32_t)kmax : 0u);
    double maxlast = okey_inv(((uint64_t)hi << 32) | lo);
    hi = w.min_u32((uint32_t)(kmin >> 32));
    lo = w.min_u32((uint32_t)(kmin >> 32) == hi ? (uint32_t)kmin : ~0u);
    double minarr = okey_inv(((uint64_t)hi << 32) | lo);
    w.sync();
    int rank = (int)ceil(0.9 * (double)n);
    if (rank < 1) rank = 1;
    lane0([&] { u().tmp_i[3] = rank - 1; });
    double p90_ttft = select_kth(p.ttft, n, rank - 1);
    lane0([&] { u().tmp_i[3] = rank - 1; });
    double p90_tpot = select_kth(p.tpot, n, rank - 1);
    if (lane == 0) {
      // Python sum(): CPython 3.12 Neumaier loop, request order
      double sums[2];
      for (int which = 0; which < 2; which++) {
        const double* v = which == 0 ? p.ttft : p.tpot;
        double f = 0.0 + v[0], cc = 0.0;
        for (int i = 1; i < n; i++) {
          double x = v[i];
          double t = f + x;
          if (fabs(f) >= fabs(x))
            cc += (f - t) + x;
          else
            cc += (x - t) + f;
          f = t;
        }
        if (cc != 0.0 && isfinite(cc)) f += cc;
        sums[which] = f;
      }
      out->n_ok = (int32_t)n_ok;
      out->attainment = (double)n_ok / (double)n;
      out->mean_ttft = sums[0] / (double)n;
      out->mean_tpot = sums[1] / (double)n;
      out->p90_ttft = p90_ttft;
      out->p90_tpot = p90_tpot;
      out->span = maxlast - minarr;
      out->goodput = out->span > 0 ? (double)n_ok / out->span : INFINITY;
    }
    w.sync();
  }

  AS_HD void finish() {
    arrow_summary_t* out = B->summaries + sid;
    const Uniform& U = sm->u;
    if (U.status == ARROW_STALLED || U.status == ARROW_INCOMPLETE) write_diag();
    if (lane == 0) {
      memset(out, 0, sizeof(*out));
      out->status = U.status;
      out->overflow = U.overflow;
      out->n_requests = sc().n_requests;
      out->n_completed = U.completed;
      out->n_flips = U.n_flips;
      out->n_events = U.n_events;
      out->n_iterations = U.n_iters;
      out->n_decisions = U.n_dec;
      out->n_ticks = U.n_ticks;
      out->n_snapshots = U.n_snap;
      out->stall_time = U.status == ARROW_STALLED ? U.stall_time : NAN;
      out->decision_hash = U.hash;
      out->n_serial_steps = U.n_serial;
      out->n_parallel_steps = U.n_rounds + U.n_bursts;
      out->cycles = clock_now() - t_start;
#if defined(ARROW_PROF) && defined(__CUDA_ARCH__)
      if (sid < ARROW_PROF_MAX)
        for (int q = 0; q < 32; q++) arrow_prof_cycles[sid * 32 + q] = U.cyc_kind[q];
#endif
      {  // profiling: per-mille of loop cycles in serial steps (high word) and rounds (low word)
        const int64_t tot = U.cyc_serial + U.cyc_round + U.cyc_burst + 1;
        out->reserved = ((U.cyc_serial * 1000 / tot) << 32) | (U.cyc_round * 1000 / tot);
      }
      out->attainment = out->p90_ttft = out->p90_tpot = NAN;
      out->mean_ttft = out->mean_tpot = out->goodput = out->span = NAN;
    }
    w.sync();
    if (U.status == ARROW_OK && sc().n_requests > 0) summarize(out);
    if (lane == 0 && U.status == ARROW_OK && U.overflow != ARROW_OVF_NONE) out->status = ARROW_BUFFER_OVERFLOW;
    // per-request outputs
    if (HAVE_OM && om.req_offset >= 0) {
      for (int r = lane; r < sc().n_requests; r += WD) {
        if (B->req_first) B->req_first[om.req_offset + r] = p.first[r];
        if (B->req_last) B->req_last[om.req_offset + r] = p.last[r];
      }
    }
    w.sync();
  }

  int64_t t_start;
  double dnow;  // event time of the last compute_delays (exact-fold fallbacks)

  AS_HD static int64_t clock_now() {
#ifdef __CUDA_ARCH__
    return (int64_t)clock64();
#else
    return 0;
#endif
  }

  AS_HD void run(int s) {
    t_start = clock_now();
    init_scenario(s);
    simulate();
    finish();
  }
};

}  // namespace arrow
