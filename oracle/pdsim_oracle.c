/*
 * pdsim_oracle.c — TEST INFRASTRUCTURE (parity checker + CPU baseline), not
 * product code.  See pdsim_oracle.h.
 *
 * A structure-preserving C restatement of the reference simulator:
 *   - the event heap keyed (time, kind, seq)          engine.py:39-45, 164-166, 267
 *   - Instance with ordered wait/running lists, FIFO migrations, parked KV,
 *     O(residents) recomputed growth/free sums           instance.py:75-390
 *   - PoolSet with insertion-ordered membership          pools.py:34-137
 *   - GlobalScheduler Alg. 1-4 + monitor triggers        scheduler.py:48-335
 *   - Monitor snapshots every tick                       monitor.py:56-73
 *   - RequestRecord / compute_metrics                    core.py:105-156, report.py:21-74
 * Nothing here is incrementalised: every helper recomputes what the
 * reference recomputes, in the same order, with the same IEEE-754 double
 * expressions (compiled with -ffp-contract=off, no fast-math).
 */
#include "pdsim_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>
#include <time.h>
#include <stdatomic.h>
#include <unistd.h>

/* ------------------------------------------------------------------ */
/* small helpers                                                      */
/* ------------------------------------------------------------------ */

#define GROW(ptr, cap, need)                                              \
  do {                                                                    \
    if ((need) > (cap)) {                                                 \
      int64_t nc_ = (cap) ? (cap) : 8;                                    \
      while (nc_ < (need)) nc_ *= 2;                                      \
      (ptr) = realloc((ptr), (size_t)nc_ * sizeof(*(ptr)));               \
      (cap) = nc_;                                                        \
    }                                                                     \
  } while (0)

/* cost_model.py:73-78 — a2 * L * L + a1 * L + a0, left to right */
static double predict_prefill(double a2, double a1, double a0, int64_t len) {
  double L = (double)len;
  return a2 * L * L + a1 * L + a0;
}

/* cost_model.py:81-85 */
static double decode_iter_time(double b1, double b0, int64_t tokens) {
  return b1 * (double)tokens + b0;
}

/* cost_model.py:88-92: prompt_len * bytes_per_token is an exact Python int */
static double transfer_time(double base, int64_t bpt, double bw, int64_t prompt) {
  return base + (double)(prompt * bpt) / bw;
}

/* CPython 3.12 builtin_sum_impl float path (Neumaier).  The first item is
 * added to the int start 0, which yields the item itself (0 + -0.0 = 0.0). */
double pdsim_oracle_pysum(const double* v, int64_t n) {
  if (n <= 0) return 0.0;
  double f = 0.0 + v[0];
  double c = 0.0;
  for (int64_t i = 1; i < n; i++) {
    double x = v[i];
    double t = f + x;
    if (fabs(f) >= fabs(x))
      c += (f - t) + x;
    else
      c += (x - t) + f;
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f += c;
  return f;
}

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* ------------------------------------------------------------------ */
/* phase requests, events                                             */
/* ------------------------------------------------------------------ */

enum { PH_PREFILL = 0, PH_DECODE = 1 };
enum { EV_MIG = 0, EV_ITER = 1, EV_PREFILL = 2, EV_ARRIVAL = 3, EV_TICK = 4 };

typedef struct preq {   /* core.PhaseRequest, core.py:70-88 */
  int rid, phase;
  int64_t prompt, out, tg, done, kv_held;
  int kv_source;        /* -1 = None */
} preq_t;

typedef struct {
  double t;
  int kind;
  int64_t seq;
  int a, b;             /* payload: instance / request / source */
} event_t;

static int ev_less(const event_t* x, const event_t* y) {
  if (x->t != y->t) return x->t < y->t;
  if (x->kind != y->kind) return x->kind < y->kind;
  return x->seq < y->seq;
}

typedef struct {
  event_t* v;
  int64_t n, cap;
} heap_t;

static void heap_push(heap_t* h, event_t e) {
  GROW(h->v, h->cap, h->n + 1);
  int64_t i = h->n++;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (!ev_less(&e, &h->v[p])) break;
    h->v[i] = h->v[p];
    i = p;
  }
  h->v[i] = e;
}

static event_t heap_pop(heap_t* h) {
  event_t top = h->v[0];
  event_t last = h->v[--h->n];
  int64_t i = 0;
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    const event_t* best = &last;
    if (l < h->n && ev_less(&h->v[l], best)) { m = l; best = &h->v[l]; }
    if (r < h->n && ev_less(&h->v[r], best)) { m = r; best = &h->v[r]; }
    if (m == i) break;
    h->v[i] = h->v[m];
    i = m;
  }
  if (h->n > 0) h->v[i] = last;
  return top;
}

/* ------------------------------------------------------------------ */
/* instance, instance.py:75-390                                        */
/* ------------------------------------------------------------------ */

typedef struct {        /* instance.BatchEntry, instance.py:54-62 */
  preq_t* req;
  int64_t tokens;
  int dedicated, completes, admit;
} entry_t;

typedef struct {
  int id;
  preq_t** wait; int64_t wait_n, wait_cap;                   /* deque, arbitrary remove */
  preq_t** mig; int64_t mig_head, mig_n, mig_cap;            /* FIFO ring */
  preq_t** run; int64_t run_n, run_cap;                      /* admission order */
  struct { int rid; int64_t tok; } *park; int64_t park_n, park_cap; /* dict rid -> tokens */
  int64_t kv_used, kv_reserved;
  int busy; double busy_until;
  entry_t* pend; int64_t pend_n, pend_cap; int has_pend;
  preq_t* active_mig;
  double* em_t; int64_t* em_k; int64_t em_head, em_n, em_cap; /* emission deque ring */
  int64_t iters;        /* begin_iteration count (for iteration-indexed outputs) */
} inst_t;

typedef struct {
  const arrow_scenario_t* sc;
  int n, N;
  int64_t kv_cap, budget, max_batch;
  double* arrival;
  const int32_t* inl;
  const int32_t* outl;
  preq_t* P;            /* prefill-phase request objects */
  preq_t* D;            /* decode-phase request objects */
  int* resident;        /* _resident_ids: instance holding the request, -1 none */
  inst_t* inst;
  /* pools.py:42-50 */
  int* pool[4]; int pool_n[4]; int* where;
  /* scheduler.py:82-85 */
  double breach;
  int64_t rr_p, rr_d;
  arrow_decision_t* dec; int64_t dec_n, dec_cap;
  int n_flips;
  /* engine.py:157-162 */
  heap_t heap;
  int64_t seq;
  int completed;
  int64_t esp;
  int64_t n_events, n_iters, n_ticks;
  /* token bookkeeping */
  double* first; double* last; int64_t* ntok;
  int32_t* req_pf; int32_t* req_dc; int32_t* req_dit;
  double* tok; const int64_t* tok_off;
  /* outputs */
  const arrow_batch_t* B;
  const arrow_outmap_t* om;
  int64_t snaps_written;
  int overflow;
  int status;
  double stall_time;
} sim_t;

static void inst_init(inst_t* I, int id) {
  memset(I, 0, sizeof(*I));
  I->id = id;
}

static void inst_free(inst_t* I) {
  free(I->wait); free(I->mig); free(I->run); free(I->park);
  free(I->pend); free(I->em_t); free(I->em_k);
}

static int fail(sim_t* S, int status) {
  if (S->status == ARROW_OK) S->status = status;
  return status;
}

/* instance.py:96-110 */
static void inst_enqueue(sim_t* S, inst_t* I, preq_t* r) {
  if (S->resident[r->rid] == I->id) { fail(S, ARROW_INTERNAL); return; }
  if (r->kv_source == I->id) { fail(S, ARROW_INTERNAL); return; }
  S->resident[r->rid] = I->id;
  if (r->phase == PH_DECODE && r->kv_source >= 0) {
    if (I->mig_n + 1 > I->mig_cap) {     /* grow ring, keep FIFO order */
      int64_t nc = I->mig_cap ? 2 * I->mig_cap : 8;
      preq_t** nv = malloc((size_t)nc * sizeof(*nv));
      for (int64_t k = 0; k < I->mig_n; k++) nv[k] = I->mig[(I->mig_head + k) % I->mig_cap];
      free(I->mig);
      I->mig = nv; I->mig_cap = nc; I->mig_head = 0;
    }
    I->mig[(I->mig_head + I->mig_n) % I->mig_cap] = r;
    I->mig_n++;
  } else {
    GROW(I->wait, I->wait_cap, I->wait_n + 1);
    I->wait[I->wait_n++] = r;
  }
}

static int64_t park_find(inst_t* I, int rid) {
  for (int64_t k = 0; k < I->park_n; k++)
    if (I->park[k].rid == rid) return k;
  return -1;
}

static int64_t park_pop(sim_t* S, inst_t* I, int rid) {
  int64_t k = park_find(I, rid);
  if (k < 0) { fail(S, ARROW_INTERNAL); return 0; }
  int64_t tok = I->park[k].tok;
  I->park[k] = I->park[I->park_n - 1];
  I->park_n--;
  return tok;
}

/* instance.py:112-118 */
static void inst_adopt_local_decode(sim_t* S, inst_t* I, preq_t* r) {
  r->kv_held = park_pop(S, I, r->rid);
  r->kv_source = -1;
  inst_enqueue(S, I, r);
}

/* instance.py:120-122 */
static void inst_release_parked(sim_t* S, inst_t* I, int rid) {
  I->kv_used -= park_pop(S, I, rid);
}

/* instance.py:159-173 */
static int64_t inst_committed_growth(inst_t* I) {
  int64_t s = 0;
  for (int64_t k = 0; k < I->run_n; k++)
    if (I->run[k]->phase == PH_DECODE) s += I->run[k]->out - 1 - I->run[k]->tg;
  return s;
}

static int64_t inst_waiting_decode_growth(inst_t* I) {
  int64_t s = 0;
  for (int64_t k = 0; k < I->wait_n; k++)
    if (I->wait[k]->phase == PH_DECODE) s += I->wait[k]->out - 1 - I->wait[k]->tg;
  return s;
}

static int64_t inst_kv_free(sim_t* S, inst_t* I) {
  return S->kv_cap - I->kv_used - I->kv_reserved - inst_committed_growth(I);
}

/* instance.py:126-146; returns 1 and sets *finish when a transfer starts */
static int inst_advance_migrations(sim_t* S, inst_t* I, double now, double* finish, preq_t** out) {
  if (I->active_mig != NULL || I->mig_n == 0) return 0;
  preq_t* r = I->mig[I->mig_head];
  int64_t need = r->prompt + (r->out - 1 - r->tg);
  if (inst_kv_free(S, I) - inst_waiting_decode_growth(I) < need) return 0;
  I->mig_head = (I->mig_head + 1) % I->mig_cap;
  I->mig_n--;
  I->kv_reserved += r->prompt;
  I->active_mig = r;
  const arrow_scenario_t* sc = S->sc;
  *finish = now + transfer_time(sc->base_latency, sc->bytes_per_token, sc->bandwidth, r->prompt);
  *out = r;
  return 1;
}

/* instance.py:148-155 */
static void inst_finish_migration(sim_t* S, inst_t* I, preq_t* r) {
  if (I->active_mig != r) { fail(S, ARROW_INTERNAL); return; }
  I->active_mig = NULL;
  I->kv_reserved -= r->prompt;
  I->kv_used += r->prompt;
  r->kv_held = r->prompt;
  GROW(I->wait, I->wait_cap, I->wait_n + 1);
  I->wait[I->wait_n++] = r;
}

static void pend_add(inst_t* I, preq_t* r, int64_t tokens, int dedicated, int completes, int admit) {
  GROW(I->pend, I->pend_cap, I->pend_n + 1);
  entry_t* e = &I->pend[I->pend_n++];
  e->req = r; e->tokens = tokens; e->dedicated = dedicated; e->completes = completes; e->admit = admit;
}

/* instance.py:175-227 — plans into I->pend (pend_n entries) */
static void inst_build_iteration_batch(sim_t* S, inst_t* I) {
  int64_t budget = S->budget;
  int64_t decode_cap = S->max_batch < budget ? S->max_batch : budget;
  int64_t kv_free = inst_kv_free(S, I);
  I->pend_n = 0;

  int64_t n_decode = 0;
  for (int64_t k = 0; k < I->run_n; k++) {
    preq_t* r = I->run[k];
    if (r->phase == PH_DECODE && n_decode < decode_cap) {
      pend_add(I, r, 1, 0, 0, 0);
      n_decode++;
    }
  }
  for (int64_t k = 0; k < I->wait_n; k++) {
    preq_t* r = I->wait[k];
    if (r->phase != PH_DECODE) continue;
    if (n_decode >= decode_cap) break;
    int64_t growth = r->out - 1 - r->tg;
    if (growth > kv_free) break;
    pend_add(I, r, 1, 0, 0, 1);
    kv_free -= growth;
    n_decode++;
  }

  int have_entries = I->pend_n > 0;
  int have_running_prefill = 0;
  for (int64_t k = 0; k < I->run_n; k++)
    if (I->run[k]->phase == PH_PREFILL) { have_running_prefill = 1; break; }
  preq_t* head = NULL;
  for (int64_t k = 0; k < I->wait_n; k++)
    if (I->wait[k]->phase == PH_PREFILL) { head = I->wait[k]; break; }

  if (!have_entries && !have_running_prefill && head != NULL) {
    if (head->done == 0 && head->prompt <= budget && head->prompt <= kv_free) {
      pend_add(I, head, head->prompt, 1, 1, 1);
      return;
    }
  }

  int64_t budget_left = budget - n_decode;
  /* running prefills (admit False) then waiting prefills (admit True) */
  for (int pass = 0; pass < 2; pass++) {
    int64_t cnt = pass == 0 ? I->run_n : I->wait_n;
    preq_t** arr = pass == 0 ? I->run : I->wait;
    for (int64_t k = 0; k < cnt; k++) {
      preq_t* r = arr[k];
      if (r->phase != PH_PREFILL) continue;
      if (budget_left <= 0) return;
      int64_t remaining = r->prompt - r->done;
      int64_t chunk = budget_left;
      if (remaining < chunk) chunk = remaining;
      if (kv_free < chunk) chunk = kv_free;
      if (chunk <= 0) return;
      pend_add(I, r, chunk, 0, chunk == remaining, pass == 1);
      budget_left -= chunk;
      kv_free -= chunk;
    }
  }
}

static void list_remove(preq_t** arr, int64_t* n, preq_t* r) {
  for (int64_t k = 0; k < *n; k++) {
    if (arr[k] == r) {
      memmove(&arr[k], &arr[k + 1], (size_t)(*n - k - 1) * sizeof(*arr));
      (*n)--;
      return;
    }
  }
}

/* instance.py:229-252 */
static double inst_begin_iteration(sim_t* S, inst_t* I, double now) {
  if (I->busy) { fail(S, ARROW_INTERNAL); return now; }
  int64_t total = 0;
  I->iters++;
  for (int64_t k = 0; k < I->pend_n; k++) {
    entry_t* e = &I->pend[k];
    total += e->tokens;
    if (e->admit) {
      list_remove(I->wait, &I->wait_n, e->req);
      GROW(I->run, I->run_cap, I->run_n + 1);
      I->run[I->run_n++] = e->req;
      if (e->req->phase == PH_DECODE && S->req_dit) S->req_dit[e->req->rid] = (int32_t)(I->iters - 1);
    }
    if (e->req->phase == PH_PREFILL) {
      I->kv_used += e->tokens;
      e->req->kv_held += e->tokens;
    }
  }
  if (I->kv_used + I->kv_reserved > S->kv_cap) fail(S, ARROW_INTERNAL);
  const arrow_scenario_t* sc = S->sc;
  double dur;
  if (I->pend[0].dedicated)
    dur = predict_prefill(sc->true_a2, sc->true_a1, sc->true_a0, I->pend[0].req->prompt);
  else
    dur = decode_iter_time(sc->b1, sc->b0, total);
  I->busy_until = now + dur;
  I->busy = 1;
  I->has_pend = 1;
  return I->busy_until;
}

typedef struct {
  int* emitted; int64_t n_emit, cap_emit;
  int* pfin; int64_t n_pfin, cap_pfin;
  int* dfin; int64_t n_dfin, cap_dfin;
} outcome_t;

/* instance.py:254-288 */
static void inst_execute_iteration(sim_t* S, inst_t* I, double now, outcome_t* o) {
  o->n_emit = o->n_pfin = o->n_dfin = 0;
  if (!I->has_pend || !I->busy || now != I->busy_until) { fail(S, ARROW_INTERNAL); return; }
  for (int64_t k = 0; k < I->pend_n; k++) {
    entry_t* e = &I->pend[k];
    preq_t* r = e->req;
    if (r->phase == PH_DECODE) {
      r->tg += 1;
      r->kv_held += 1;
      I->kv_used += 1;
      GROW(o->emitted, o->cap_emit, o->n_emit + 1);
      o->emitted[o->n_emit++] = r->rid;
      if (r->tg == r->out - 1) {
        I->kv_used -= r->kv_held;
        list_remove(I->run, &I->run_n, r);
        if (S->resident[r->rid] == I->id) S->resident[r->rid] = -1;
        GROW(o->dfin, o->cap_dfin, o->n_dfin + 1);
        o->dfin[o->n_dfin++] = r->rid;
      }
    } else {
      r->done += e->tokens;
      if (e->completes) {
        if (r->done != r->prompt) { fail(S, ARROW_INTERNAL); return; }
        list_remove(I->run, &I->run_n, r);
        if (S->resident[r->rid] == I->id) S->resident[r->rid] = -1;
        GROW(I->park, I->park_cap, I->park_n + 1);
        int64_t kk = park_find(I, r->rid);
        if (kk < 0) { kk = I->park_n++; I->park[kk].rid = r->rid; }
        I->park[kk].tok = r->kv_held;
        GROW(o->pfin, o->cap_pfin, o->n_pfin + 1);
        o->pfin[o->n_pfin++] = r->rid;
      }
    }
  }
  I->has_pend = 0;
  I->pend_n = 0;
  I->busy = 0;
  int64_t ntok = o->n_emit + o->n_pfin;
  if (ntok) {
    if (I->em_n + 1 > I->em_cap) {
      int64_t nc = I->em_cap ? 2 * I->em_cap : 64;
      double* nt = malloc((size_t)nc * sizeof(double));
      int64_t* nk = malloc((size_t)nc * sizeof(int64_t));
      for (int64_t k = 0; k < I->em_n; k++) {
        nt[k] = I->em_t[(I->em_head + k) % I->em_cap];
        nk[k] = I->em_k[(I->em_head + k) % I->em_cap];
      }
      free(I->em_t); free(I->em_k);
      I->em_t = nt; I->em_k = nk; I->em_cap = nc; I->em_head = 0;
    }
    I->em_t[(I->em_head + I->em_n) % I->em_cap] = now;
    I->em_k[(I->em_head + I->em_n) % I->em_cap] = ntok;
    I->em_n++;
    double horizon = now - 2 * S->sc->window;
    while (I->em_n > 0 && I->em_t[I->em_head] < horizon) {
      I->em_head = (I->em_head + 1) % I->em_cap;
      I->em_n--;
    }
  }
}

/* instance.py:292-302 */
static int64_t inst_running_tokens(inst_t* I) {
  int64_t total = 0;
  for (int64_t k = 0; k < I->run_n; k++)
    if (I->run[k]->phase == PH_DECODE) total += I->run[k]->prompt + I->run[k]->tg;
  for (int64_t k = 0; k < I->wait_n; k++)
    if (I->wait[k]->phase == PH_DECODE) total += I->wait[k]->prompt + I->wait[k]->tg;
  return total;
}

/* instance.py:304-321 */
static double inst_predicted_prefill_delay(sim_t* S, inst_t* I, double now) {
  const arrow_scenario_t* sc = S->sc;
  double delay = 0.0;
  if (I->busy) {
    double x = I->busy_until - now;
    delay += (0.0 > x) ? 0.0 : x;    /* Python max(x, 0.0) keeps x unless 0.0 > x */
  }
  for (int64_t k = 0; k < I->run_n; k++)
    if (I->run[k]->phase == PH_PREFILL)
      delay += predict_prefill(sc->pred_a2, sc->pred_a1, sc->pred_a0, I->run[k]->prompt - I->run[k]->done);
  for (int64_t k = 0; k < I->wait_n; k++)
    if (I->wait[k]->phase == PH_PREFILL)
      delay += predict_prefill(sc->pred_a2, sc->pred_a1, sc->pred_a0, I->wait[k]->prompt - I->wait[k]->done);
  return delay;
}

/* instance.py:323-329; returns 0 for None */
static int inst_avg_token_interval(inst_t* I, double window, double now, double* out) {
  double lo = now - window;
  int64_t cnt = 0;
  double first = 0.0, lastv = 0.0;
  for (int64_t k = 0; k < I->em_n; k++) {
    double t = I->em_t[(I->em_head + k) % I->em_cap];
    if (t >= lo) {
      if (cnt == 0) first = t;
      lastv = t;
      cnt++;
    }
  }
  if (cnt < 2) return 0;
  *out = (lastv - first) / (double)(cnt - 1);
  return 1;
}

/* instance.py:333-360 */
static int inst_has_prefill_work(inst_t* I) {
  for (int64_t k = 0; k < I->run_n; k++) if (I->run[k]->phase == PH_PREFILL) return 1;
  for (int64_t k = 0; k < I->wait_n; k++) if (I->wait[k]->phase == PH_PREFILL) return 1;
  return 0;
}

static int inst_has_decode_work(inst_t* I) {
  if (I->active_mig != NULL || I->mig_n > 0) return 1;
  for (int64_t k = 0; k < I->run_n; k++) if (I->run[k]->phase == PH_DECODE) return 1;
  for (int64_t k = 0; k < I->wait_n; k++) if (I->wait[k]->phase == PH_DECODE) return 1;
  return 0;
}

static int inst_has_startable_work(inst_t* I) { return I->run_n > 0 || I->wait_n > 0; }

static int64_t inst_prefill_queue_len(inst_t* I) {
  int64_t c = 0;
  for (int64_t k = 0; k < I->wait_n; k++) c += I->wait[k]->phase == PH_PREFILL;
  return c;
}

static int64_t inst_prefill_count(inst_t* I) {
  int64_t c = 0;
  for (int64_t k = 0; k < I->run_n; k++) c += I->run[k]->phase == PH_PREFILL;
  return c + inst_prefill_queue_len(I);
}

static int64_t inst_decode_count(inst_t* I) {
  int64_t c = 0;
  for (int64_t k = 0; k < I->run_n; k++) c += I->run[k]->phase == PH_DECODE;
  for (int64_t k = 0; k < I->wait_n; k++) c += I->wait[k]->phase == PH_DECODE;
  c += I->mig_n;
  if (I->active_mig != NULL) c += 1;
  return c;
}

/* instance.py:380-390 */
static int inst_idle_and_empty(inst_t* I) {
  return !I->busy && I->run_n == 0 && I->wait_n == 0 && I->mig_n == 0 && I->active_mig == NULL &&
         I->park_n == 0 && I->kv_used == 0 && I->kv_reserved == 0;
}

/* ------------------------------------------------------------------ */
/* pools, pools.py:34-137                                             */
/* ------------------------------------------------------------------ */

static const int LEGAL[4][4] = {
    /* from PREFILL */ {0, 1, 1, 0},   /* -> DECODE, P_TO_D */
    /* from DECODE  */ {1, 0, 0, 1},   /* -> PREFILL, D_TO_P */
    /* from P_TO_D  */ {1, 1, 0, 0},   /* -> PREFILL, DECODE */
    /* from D_TO_P  */ {1, 1, 0, 0},   /* -> PREFILL, DECODE */
};

static int pool_move(sim_t* S, int id, int to) {   /* pools.py:76-85 */
  int src = S->where[id];
  if (!LEGAL[src][to]) { fail(S, ARROW_INTERNAL); return src; }
  int* m = S->pool[src];
  for (int k = 0; k < S->pool_n[src]; k++) {
    if (m[k] == id) {
      memmove(&m[k], &m[k + 1], (size_t)(S->pool_n[src] - k - 1) * sizeof(int));
      S->pool_n[src]--;
      break;
    }
  }
  S->pool[to][S->pool_n[to]++] = id;
  S->where[id] = to;
  return to;
}

/* pools.py:87-102; -1 = None */
static int flip_to_decode_role(sim_t* S, int id, int has_prefill_work) {
  int src = S->where[id];
  if (src == ARROW_POOL_DECODE || src == ARROW_POOL_P_TO_D) return -1;
  if (src == ARROW_POOL_PREFILL)
    return pool_move(S, id, has_prefill_work ? ARROW_POOL_P_TO_D : ARROW_POOL_DECODE);
  return pool_move(S, id, ARROW_POOL_DECODE);
}

/* pools.py:104-114 */
static int flip_to_prefill_role(sim_t* S, int id, int has_decode_work) {
  int src = S->where[id];
  if (src == ARROW_POOL_PREFILL || src == ARROW_POOL_D_TO_P) return -1;
  if (src == ARROW_POOL_DECODE)
    return pool_move(S, id, has_decode_work ? ARROW_POOL_D_TO_P : ARROW_POOL_PREFILL);
  return pool_move(S, id, ARROW_POOL_PREFILL);
}

/* pools.py:116-123 */
static int pool_on_drained(sim_t* S, int id, int drained_phase) {
  int src = S->where[id];
  if (src == ARROW_POOL_P_TO_D && drained_phase == PH_PREFILL) return pool_move(S, id, ARROW_POOL_DECODE);
  if (src == ARROW_POOL_D_TO_P && drained_phase == PH_DECODE) return pool_move(S, id, ARROW_POOL_PREFILL);
  return -1;
}

/* ------------------------------------------------------------------ */
/* scheduler, scheduler.py:48-335                                     */
/* ------------------------------------------------------------------ */

static void log_decision(sim_t* S, double now, int kind, int rid, int inst, int code) {
  GROW(S->dec, S->dec_cap, S->dec_n + 1);
  arrow_decision_t* d = &S->dec[S->dec_n++];
  d->time = now;
  d->request = rid;
  d->instance = (int16_t)inst;
  d->kind = (uint8_t)kind;
  d->code = (uint8_t)code;
}

static void log_dispatch(sim_t* S, double now, int kind, int rid, int inst, int branch) {
  log_decision(S, now, kind, rid, inst, branch);
  if (kind == ARROW_DEC_PREFILL_DISPATCH) {
    if (S->req_pf) S->req_pf[rid] = inst | (branch << 16);
  } else {
    if (S->req_dc) S->req_dc[rid] = inst | (branch << 16);
  }
}

static void log_flip(sim_t* S, double now, int inst, int src, int dst, int trigger) {
  log_decision(S, now, ARROW_DEC_FLIP, -1, inst, trigger | (src << 3) | (dst << 5));
  S->n_flips++;
}

/* _argmin over a member list with a float key (delay); -1 = None */
static int argmin_delay(sim_t* S, const int* ids, int n, double now, double* best_val) {
  int best = -1;
  double bv = 0.0;
  for (int k = 0; k < n; k++) {
    double v = inst_predicted_prefill_delay(S, &S->inst[ids[k]], now);
    if (best < 0 || v < bv) { best = ids[k]; bv = v; }
  }
  *best_val = bv;
  return best;
}

static int argmin_tokens(sim_t* S, const int* ids, int n, int64_t* best_val) {
  int best = -1;
  int64_t bv = 0;
  for (int k = 0; k < n; k++) {
    int64_t v = inst_running_tokens(&S->inst[ids[k]]);
    if (best < 0 || v < bv) { best = ids[k]; bv = v; }
  }
  *best_val = bv;
  return best;
}

/* members(DECODE) + members(P_TO_D) into buf; returns count */
static int decode_role_ids(sim_t* S, int* buf) {
  int c = 0;
  for (int k = 0; k < S->pool_n[ARROW_POOL_DECODE]; k++) buf[c++] = S->pool[ARROW_POOL_DECODE][k];
  for (int k = 0; k < S->pool_n[ARROW_POOL_P_TO_D]; k++) buf[c++] = S->pool[ARROW_POOL_P_TO_D][k];
  return c;
}

/* scheduler.py:124-134; 0 = None */
static int pool_mean_interval(sim_t* S, double now, double* out) {
  int ids[128];
  double vals[128];
  int n = decode_role_ids(S, ids), m = 0;
  for (int k = 0; k < n; k++) {
    double v;
    if (inst_avg_token_interval(&S->inst[ids[k]], S->sc->window, now, &v)) vals[m++] = v;
  }
  if (m == 0) return 0;
  *out = pdsim_oracle_pysum(vals, m) / (double)m;
  return 1;
}

/* scheduler.py:136-147 */
static int decode_load_is_low(sim_t* S, double now) {
  int ids[128];
  int n = decode_role_ids(S, ids);
  if (n == 0) return 0;
  int64_t min_tokens;
  argmin_tokens(S, ids, n, &min_tokens);
  if ((double)min_tokens > S->sc->theta_d * (double)S->sc->max_tokens) return 0;
  double mean;
  if (!pool_mean_interval(S, now, &mean)) return 1;
  return mean <= S->sc->tpot_thr;
}

/* scheduler.py:258-276 */
static int try_move_decode_to_prefill(sim_t* S, double now, int trigger) {
  if (!S->sc->enable_flips) return -1;
  if (S->pool_n[ARROW_POOL_DECODE] + S->pool_n[ARROW_POOL_P_TO_D] <= 1) return -1;
  int ids[128];
  int n = S->pool_n[ARROW_POOL_P_TO_D];
  if (n > 0) memcpy(ids, S->pool[ARROW_POOL_P_TO_D], (size_t)n * sizeof(int));
  else { n = S->pool_n[ARROW_POOL_DECODE]; memcpy(ids, S->pool[ARROW_POOL_DECODE], (size_t)n * sizeof(int)); }
  int64_t tv;
  int chosen = argmin_tokens(S, ids, n, &tv);
  inst_t* I = &S->inst[chosen];
  int src = S->where[chosen];
  int dst = flip_to_prefill_role(S, chosen, inst_has_decode_work(I));
  if (dst < 0) return -1;
  log_flip(S, now, chosen, src, dst, trigger);
  return chosen;
}

/* scheduler.py:278-296 */
static int try_move_prefill_to_decode(sim_t* S, double now, int trigger) {
  if (!S->sc->enable_flips) return -1;
  if (S->pool_n[ARROW_POOL_PREFILL] + S->pool_n[ARROW_POOL_D_TO_P] <= 1) return -1;
  int ids[128];
  int n = S->pool_n[ARROW_POOL_D_TO_P];
  if (n > 0) memcpy(ids, S->pool[ARROW_POOL_D_TO_P], (size_t)n * sizeof(int));
  else { n = S->pool_n[ARROW_POOL_PREFILL]; memcpy(ids, S->pool[ARROW_POOL_PREFILL], (size_t)n * sizeof(int)); }
  double dv;
  int chosen = argmin_delay(S, ids, n, now, &dv);
  inst_t* I = &S->inst[chosen];
  int src = S->where[chosen];
  int dst = flip_to_decode_role(S, chosen, inst_has_prefill_work(I));
  if (dst < 0) return -1;
  log_flip(S, now, chosen, src, dst, trigger);
  return chosen;
}

/* scheduler.py:151-195 */
static int schedule_prefill(sim_t* S, int rid, double now) {
  const arrow_scenario_t* sc = S->sc;
  const int K = ARROW_DEC_PREFILL_DISPATCH;
  if (sc->strategy == ARROW_STRATEGY_ROUND_ROBIN) {
    int n = S->pool_n[ARROW_POOL_PREFILL];
    int chosen = S->pool[ARROW_POOL_PREFILL][S->rr_p % n];
    S->rr_p++;
    log_dispatch(S, now, K, rid, chosen, ARROW_BR_ROUND_ROBIN);
    return chosen;
  }
  if (sc->strategy == ARROW_STRATEGY_MINIMAL_LOAD) {
    double dv;
    int chosen = argmin_delay(S, S->pool[ARROW_POOL_PREFILL], S->pool_n[ARROW_POOL_PREFILL], now, &dv);
    log_dispatch(S, now, K, rid, chosen, ARROW_BR_MIN_LOAD);
    return chosen;
  }
  double own = predict_prefill(sc->pred_a2, sc->pred_a1, sc->pred_a0, S->inl[rid]);
  double d1, d2;
  int t1 = argmin_delay(S, S->pool[ARROW_POOL_PREFILL], S->pool_n[ARROW_POOL_PREFILL], now, &d1);
  if (t1 >= 0 && d1 + own <= sc->ttft_thr) { log_dispatch(S, now, K, rid, t1, ARROW_BR_ALG1_T1); return t1; }
  int t2 = argmin_delay(S, S->pool[ARROW_POOL_D_TO_P], S->pool_n[ARROW_POOL_D_TO_P], now, &d2);
  if (t2 >= 0 && d2 + own <= sc->ttft_thr) { log_dispatch(S, now, K, rid, t2, ARROW_BR_ALG1_T2); return t2; }
  if (sc->enable_flips && decode_load_is_low(S, now)) {
    int t3 = try_move_decode_to_prefill(S, now, ARROW_TRIG_ALG1);
    if (t3 >= 0) { log_dispatch(S, now, K, rid, t3, ARROW_BR_ALG1_FLIP); return t3; }
  }
  if (t1 >= 0) { log_dispatch(S, now, K, rid, t1, ARROW_BR_ALG1_FALLBACK); return t1; }
  if (t2 >= 0) { log_dispatch(S, now, K, rid, t2, ARROW_BR_ALG1_FALLBACK); return t2; }
  int ids[128];
  int n = decode_role_ids(S, ids);
  double dv;
  int chosen = argmin_delay(S, ids, n, now, &dv);
  if (chosen < 0) { fail(S, ARROW_NO_INSTANCE); return -1; }
  log_dispatch(S, now, K, rid, chosen, ARROW_BR_ALG1_DEGENERATE);
  return chosen;
}

/* scheduler.py:214-218 */
static int decode_admissible(sim_t* S, int id, int64_t tokens, double now) {
  if (tokens > S->sc->max_tokens) return 0;
  double v;
  if (!inst_avg_token_interval(&S->inst[id], S->sc->window, now, &v)) return 1;
  return v <= S->sc->tpot_thr;
}

/* scheduler.py:199-254 */
static int schedule_decode(sim_t* S, int rid, int src, double now) {
  const arrow_scenario_t* sc = S->sc;
  const int K = ARROW_DEC_DECODE_DISPATCH;
  if (sc->strategy == ARROW_STRATEGY_ROUND_ROBIN) {
    int n = S->pool_n[ARROW_POOL_DECODE];
    int chosen = S->pool[ARROW_POOL_DECODE][S->rr_d % n];
    S->rr_d++;
    log_dispatch(S, now, K, rid, chosen, ARROW_BR_ROUND_ROBIN);
    return chosen;
  }
  if (sc->strategy == ARROW_STRATEGY_MINIMAL_LOAD) {
    int64_t tv;
    int chosen = argmin_tokens(S, S->pool[ARROW_POOL_DECODE], S->pool_n[ARROW_POOL_DECODE], &tv);
    log_dispatch(S, now, K, rid, chosen, ARROW_BR_MIN_LOAD);
    return chosen;
  }
  int sp = S->where[src];
  if (sp == ARROW_POOL_DECODE || sp == ARROW_POOL_P_TO_D) {
    log_dispatch(S, now, K, rid, src, ARROW_BR_ALG2_ZERO_TRANSFER);
    return src;
  }
  int64_t tok1, tok2;
  int t1 = argmin_tokens(S, S->pool[ARROW_POOL_DECODE], S->pool_n[ARROW_POOL_DECODE], &tok1);
  if (t1 >= 0 && decode_admissible(S, t1, tok1, now)) { log_dispatch(S, now, K, rid, t1, ARROW_BR_ALG2_T1); return t1; }
  int t2 = argmin_tokens(S, S->pool[ARROW_POOL_P_TO_D], S->pool_n[ARROW_POOL_P_TO_D], &tok2);
  if (t2 >= 0 && decode_admissible(S, t2, tok2, now)) { log_dispatch(S, now, K, rid, t2, ARROW_BR_ALG2_T2); return t2; }
  if (sc->enable_flips) {
    int t3 = try_move_prefill_to_decode(S, now, ARROW_TRIG_ALG2);
    if (t3 >= 0) { log_dispatch(S, now, K, rid, t3, ARROW_BR_ALG2_FLIP); return t3; }
  }
  if (t1 >= 0 && (t2 < 0 || tok1 <= tok2)) { log_dispatch(S, now, K, rid, t1, ARROW_BR_ALG2_FALLBACK); return t1; }
  if (t2 >= 0) { log_dispatch(S, now, K, rid, t2, ARROW_BR_ALG2_FALLBACK); return t2; }
  log_dispatch(S, now, K, rid, src, ARROW_BR_ALG2_FORCED_LOCAL);
  return src;
}

/* scheduler.py:300-335 */
static void scheduler_monitor_tick(sim_t* S, double now) {
  const arrow_scenario_t* sc = S->sc;
  if (sc->strategy != ARROW_STRATEGY_SLO_AWARE || !sc->enable_flips) return;
  double mean;
  if (pool_mean_interval(S, now, &mean) && mean > sc->tpot_thr) {
    S->breach += sc->monitor_period;
    if (S->breach >= sc->breach_duration) try_move_prefill_to_decode(S, now, ARROW_TRIG_MONITOR_TPOT);
  } else {
    S->breach = 0.0;
  }
  int ids[128];
  int n = decode_role_ids(S, ids);
  if (n == 0) return;
  int64_t aggregate = 0;
  for (int k = 0; k < n; k++) aggregate += inst_running_tokens(&S->inst[ids[k]]);
  int64_t capacity = sc->max_tokens * (int64_t)n;
  if (capacity == 0) { fail(S, ARROW_ZERO_DIVISION); return; }
  if ((double)aggregate / (double)capacity <= sc->theta_busy) return;
  int snap[128];
  int np = S->pool_n[ARROW_POOL_PREFILL];
  memcpy(snap, S->pool[ARROW_POOL_PREFILL], (size_t)np * sizeof(int));
  for (int k = 0; k < np; k++) {
    if (S->pool_n[ARROW_POOL_PREFILL] + S->pool_n[ARROW_POOL_D_TO_P] <= 1) break;
    inst_t* I = &S->inst[snap[k]];
    if (inst_has_prefill_work(I) || I->busy) continue;
    int src = S->where[snap[k]];
    int dst = flip_to_decode_role(S, snap[k], 0);
    if (dst >= 0) log_flip(S, now, snap[k], src, dst, ARROW_TRIG_MONITOR_IDLE);
  }
}

/* ------------------------------------------------------------------ */
/* engine, engine.py:122-316                                          */
/* ------------------------------------------------------------------ */

static void push(sim_t* S, double t, int kind, int a, int b) {
  event_t e = {t, kind, S->seq, a, b};
  heap_push(&S->heap, e);
  S->seq++;
}

static void add_token(sim_t* S, int rid, double now) {
  if (S->ntok[rid] == 0) S->first[rid] = now;
  S->last[rid] = now;
  if (S->tok) S->tok[S->tok_off[rid] + S->ntok[rid]] = now;
  S->ntok[rid]++;
}

static void kick(sim_t* S, inst_t* I, double now) {       /* engine.py:170-177 */
  if (I->busy || !inst_has_startable_work(I)) return;
  inst_build_iteration_batch(S, I);
  if (I->pend_n == 0) return;
  double finish = inst_begin_iteration(S, I, now);
  push(S, finish, EV_ITER, I->id, 0);
}

static void start_migrations(sim_t* S, inst_t* I, double now) {  /* engine.py:179-181 */
  double finish;
  preq_t* r;
  if (inst_advance_migrations(S, I, now, &finish, &r)) push(S, finish, EV_MIG, I->id, r->rid);
}

static void check_drained(sim_t* S, inst_t* I, double now) {    /* engine.py:183-192 */
  int kind = S->where[I->id];
  if (kind == ARROW_POOL_P_TO_D && !inst_has_prefill_work(I)) {
    int dst = pool_on_drained(S, I->id, PH_PREFILL);
    if (dst >= 0) log_flip(S, now, I->id, kind, dst, ARROW_TRIG_DRAINED);
  } else if (kind == ARROW_POOL_D_TO_P && !inst_has_decode_work(I)) {
    int dst = pool_on_drained(S, I->id, PH_DECODE);
    if (dst >= 0) log_flip(S, now, I->id, kind, dst, ARROW_TRIG_DRAINED);
  }
}

static void complete_request(sim_t* S) {                        /* engine.py:194-196 */
  S->completed++;
  S->esp = 0;
}

static void on_arrival(sim_t* S, double now, int rid) {         /* engine.py:198-203 */
  preq_t* r = &S->P[rid];
  int target = schedule_prefill(S, rid, now);
  if (target < 0) return;
  inst_t* I = &S->inst[target];
  inst_enqueue(S, I, r);
  kick(S, I, now);
}

static void on_iteration_complete(sim_t* S, double now, int id, outcome_t* o) {   /* engine.py:205-223 */
  inst_t* I = &S->inst[id];
  S->n_iters++;
  if (S->B->iterlog && S->om && S->om->iterlog_offset >= 0) {
    int64_t it = I->iters - 1;
    if (it < S->om->iterlog_stride)
      S->B->iterlog[S->om->iterlog_offset + (int64_t)id * S->om->iterlog_stride + it] = now;
    else if (S->overflow == ARROW_OVF_NONE)
      S->overflow = ARROW_OVF_ITERLOG;
  }
  inst_execute_iteration(S, I, now, o);
  if (o->n_emit || o->n_pfin) S->esp = 0;
  for (int64_t k = 0; k < o->n_emit; k++) add_token(S, o->emitted[k], now);
  for (int64_t k = 0; k < o->n_pfin; k++) {
    int rid = o->pfin[k];
    add_token(S, rid, now);
    if (S->outl[rid] == 1) {
      inst_release_parked(S, I, rid);
      complete_request(S);
    } else {
      push(S, now, EV_PREFILL, rid, id);
    }
  }
  for (int64_t k = 0; k < o->n_dfin; k++) complete_request(S);
  check_drained(S, I, now);
  start_migrations(S, I, now);
  kick(S, I, now);
}

static void on_prefill_complete(sim_t* S, double now, int rid, int src) {    /* engine.py:225-236 */
  preq_t* d = &S->D[rid];
  int target = schedule_decode(S, rid, src, now);
  inst_t* I = &S->inst[target];
  if (target == src) {
    inst_adopt_local_decode(S, I, d);
  } else {
    d->kv_source = src;
    inst_enqueue(S, I, d);
    start_migrations(S, I, now);
  }
  kick(S, I, now);
}

static void on_migration_complete(sim_t* S, double now, int id, int rid) {   /* engine.py:238-248 */
  inst_t* I = &S->inst[id];
  preq_t* d = &S->D[rid];
  inst_finish_migration(S, I, d);
  inst_t* src = &S->inst[d->kv_source];
  inst_release_parked(S, src, rid);
  start_migrations(S, I, now);
  start_migrations(S, src, now);
  kick(S, I, now);
  kick(S, src, now);
}

static void on_monitor_tick(sim_t* S, double now) {             /* engine.py:250-255 */
  const arrow_batch_t* B = S->B;
  S->n_ticks++;
  /* Monitor.collect, monitor.py:56-73 (computed every tick, as the reference does) */
  for (int i = 0; i < S->N; i++) {
    inst_t* I = &S->inst[i];
    arrow_snapshot_t s;
    double iv;
    s.time = now;
    s.instance = i;
    s.pool = S->where[i];
    s.running_tokens = (int32_t)inst_running_tokens(I);
    s.kv_used = (int32_t)I->kv_used;
    s.queue_len = (int32_t)inst_prefill_queue_len(I);
    s.pred_delay = inst_predicted_prefill_delay(S, I, now);
    s.avg_interval = inst_avg_token_interval(I, S->sc->window, now, &iv) ? iv : NAN;
    s.prefill_count = (int32_t)inst_prefill_count(I);
    s.decode_count = (int32_t)inst_decode_count(I);
    s.reserved = 0;
    if (B->snapshots && S->om && S->om->snapshot_offset >= 0) {
      if (S->snaps_written < S->om->snapshot_capacity)
        B->snapshots[S->om->snapshot_offset + S->snaps_written] = s;
      else if (S->overflow == ARROW_OVF_NONE)
        S->overflow = ARROW_OVF_SNAPSHOTS;
      S->snaps_written++;
    }
  }
  scheduler_monitor_tick(S, now);
  if (S->completed < S->n) push(S, now + S->sc->monitor_period, EV_TICK, 0, 0);
}

static void write_diag(sim_t* S) {                               /* engine.py:305-316 */
  const arrow_batch_t* B = S->B;
  if (!B->diag || !S->om || S->om->diag_offset < 0) return;
  for (int i = 0; i < S->N; i++) {
    inst_t* I = &S->inst[i];
    arrow_instdiag_t* d = &B->diag[S->om->diag_offset + i];
    d->busy_until = I->busy ? I->busy_until : NAN;
    d->pool = S->where[i];
    d->kv_used = (int32_t)I->kv_used;
    d->running = (int32_t)I->run_n;
    d->waiting = (int32_t)I->wait_n;
    d->migrating = (int32_t)I->mig_n;
    d->reserved = 0;
  }
}

static uint64_t fnv_mix(uint64_t h, uint64_t w) { return (h ^ w) * 1099511628211ULL; }

uint64_t pdsim_oracle_decision_hash(const arrow_decision_t* d, int64_t n) {
  uint64_t h = 14695981039346656037ULL;
  for (int64_t k = 0; k < n; k++) {
    uint64_t tb;
    memcpy(&tb, &d[k].time, 8);
    h = fnv_mix(h, tb);
    h = fnv_mix(h, (uint64_t)d[k].kind | ((uint64_t)d[k].code << 8) |
                       ((uint64_t)(uint16_t)d[k].instance << 16) |
                       ((uint64_t)(uint32_t)d[k].request << 32));
  }
  return h;
}

static void simulate(sim_t* S) {                                  /* engine.py:259-303 */
  outcome_t o;
  memset(&o, 0, sizeof(o));
  for (int rid = 0; rid < S->n; rid++) push(S, S->arrival[rid], EV_ARRIVAL, rid, 0);
  if (S->n > 0) push(S, S->sc->monitor_period, EV_TICK, 0, 0);
  while (S->heap.n > 0 && S->status == ARROW_OK) {
    event_t e = heap_pop(&S->heap);
    double now = e.t;
    S->esp++;
    S->n_events++;
    switch (e.kind) {
      case EV_MIG: on_migration_complete(S, now, e.a, e.b); break;
      case EV_ITER: on_iteration_complete(S, now, e.a, &o); break;
      case EV_PREFILL: on_prefill_complete(S, now, e.a, e.b); break;
      case EV_ARRIVAL: on_arrival(S, now, e.a); break;
      default: on_monitor_tick(S, now); break;
    }
    if (S->status != ARROW_OK) break;
    if (S->esp > S->sc->stall_limit) {
      S->status = ARROW_STALLED;
      S->stall_time = now;
      write_diag(S);
      break;
    }
  }
  free(o.emitted); free(o.pfin); free(o.dfin);
  if (S->status != ARROW_OK) return;
  if (S->completed != S->n) {
    S->status = ARROW_INCOMPLETE;
    S->stall_time = NAN;
    write_diag(S);
    return;
  }
  for (int i = 0; i < S->N; i++)
    if (!inst_idle_and_empty(&S->inst[i])) { S->status = ARROW_NOT_DRAINED; return; }
}

/* report.py:55-74 over RequestRecord.from_token_times (core.py:105-156) */
static void summarize(sim_t* S, arrow_summary_t* out) {
  int n = S->n;
  const arrow_scenario_t* sc = S->sc;
  double* ttft = malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  double* tpot = malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  int n_ok = 0;
  double maxlast = -INFINITY, minarr = INFINITY;
  for (int r = 0; r < n; r++) {
    double a = S->arrival[r];
    ttft[r] = S->first[r] - a;
    int64_t m = S->ntok[r];
    tpot[r] = m == 1 ? 0.0 : (S->last[r] - S->first[r]) / (double)(m - 1);
    int ok = (ttft[r] <= sc->ttft_slo) && (tpot[r] <= sc->tpot_slo);
    n_ok += ok;
    if (S->last[r] > maxlast) maxlast = S->last[r];
    if (a < minarr) minarr = a;
  }
  out->n_ok = n_ok;
  if (n > 0) {
    out->attainment = (double)n_ok / (double)n;
    out->mean_ttft = pdsim_oracle_pysum(ttft, n) / (double)n;
    out->mean_tpot = pdsim_oracle_pysum(tpot, n) / (double)n;
    int64_t rank = (int64_t)ceil(0.9 * (double)n);
    if (rank < 1) rank = 1;
    qsort(ttft, (size_t)n, sizeof(double), cmp_double);
    qsort(tpot, (size_t)n, sizeof(double), cmp_double);
    out->p90_ttft = ttft[rank - 1];
    out->p90_tpot = tpot[rank - 1];
    out->span = maxlast - minarr;
    out->goodput = out->span > 0 ? (double)n_ok / out->span : INFINITY;
  }
  free(ttft);
  free(tpot);
}

int pdsim_oracle_run_one(const arrow_batch_t* B, int s) {
  const arrow_scenario_t* sc = &B->scenarios[s];
  arrow_summary_t* sum = &B->summaries[s];
  const arrow_outmap_t* om = B->outmap ? &B->outmap[s] : NULL;
  sim_t S;
  memset(&S, 0, sizeof(S));
  S.sc = sc;
  S.B = B;
  S.om = om;
  S.n = sc->n_requests;
  S.N = sc->n_instances;
  S.kv_cap = sc->kv_capacity;
  S.budget = sc->chunk_budget;
  S.max_batch = sc->max_batch;
  S.status = ARROW_OK;
  S.stall_time = NAN;
  int n = S.n, N = S.N;
  size_t nn = (size_t)(n > 0 ? n : 1);
  S.inl = B->input_len + sc->trace_offset;
  S.outl = B->output_len + sc->trace_offset;
  S.arrival = malloc(nn * sizeof(double));
  for (int r = 0; r < n; r++) S.arrival[r] = B->arrival[sc->trace_offset + r] * sc->arrival_scale;
  S.P = calloc(nn, sizeof(preq_t));
  S.D = calloc(nn, sizeof(preq_t));
  S.resident = malloc(nn * sizeof(int));
  S.first = malloc(nn * sizeof(double));
  S.last = malloc(nn * sizeof(double));
  S.ntok = calloc(nn, sizeof(int64_t));
  int64_t* tok_off = NULL;
  for (int r = 0; r < n; r++) {
    preq_t* p = &S.P[r];
    p->rid = r; p->phase = PH_PREFILL; p->prompt = S.inl[r]; p->out = S.outl[r]; p->kv_source = -1;
    preq_t* d = &S.D[r];
    d->rid = r; d->phase = PH_DECODE; d->prompt = S.inl[r]; d->out = S.outl[r]; d->kv_source = -1;
    S.resident[r] = -1;
    S.first[r] = NAN;
    S.last[r] = NAN;
  }
  if (om && om->req_offset >= 0) {
    if (B->req_prefill) { S.req_pf = B->req_prefill + om->req_offset; for (int r = 0; r < n; r++) S.req_pf[r] = -1; }
    if (B->req_decode) { S.req_dc = B->req_decode + om->req_offset; for (int r = 0; r < n; r++) S.req_dc[r] = -1; }
    if (B->req_decode_iter) { S.req_dit = B->req_decode_iter + om->req_offset; for (int r = 0; r < n; r++) S.req_dit[r] = -1; }
  }
  if (om && om->token_offset >= 0 && B->token_times) {
    tok_off = malloc(nn * sizeof(int64_t));
    int64_t acc = om->token_offset;
    for (int r = 0; r < n; r++) { tok_off[r] = acc; acc += S.outl[r]; }
    S.tok = B->token_times;
    S.tok_off = tok_off;
  }
  S.inst = calloc((size_t)N, sizeof(inst_t));
  S.where = malloc((size_t)N * sizeof(int));
  for (int k = 0; k < 4; k++) S.pool[k] = malloc((size_t)N * sizeof(int));
  for (int i = 0; i < N; i++) {
    inst_init(&S.inst[i], i);
    int kind = i < sc->n_prefill_init ? ARROW_POOL_PREFILL : ARROW_POOL_DECODE;
    S.pool[kind][S.pool_n[kind]++] = i;
    S.where[i] = kind;
  }

  simulate(&S);

  memset(sum, 0, sizeof(*sum));
  sum->status = S.status;
  sum->overflow = S.overflow;
  sum->n_requests = n;
  sum->n_completed = S.completed;
  sum->n_flips = S.n_flips;
  sum->n_events = S.n_events;
  sum->n_iterations = S.n_iters;
  sum->n_decisions = S.dec_n;
  sum->n_ticks = S.n_ticks;
  sum->n_snapshots = S.snaps_written;
  sum->stall_time = S.stall_time;
  sum->decision_hash = pdsim_oracle_decision_hash(S.dec, S.dec_n);
  sum->attainment = sum->p90_ttft = sum->p90_tpot = NAN;
  sum->mean_ttft = sum->mean_tpot = sum->goodput = sum->span = NAN;
  if (S.status == ARROW_OK) summarize(&S, sum);
  if (S.overflow != ARROW_OVF_NONE && S.status == ARROW_OK) sum->status = ARROW_BUFFER_OVERFLOW;

  if (om && om->req_offset >= 0) {
    if (B->req_first) memcpy(B->req_first + om->req_offset, S.first, (size_t)n * sizeof(double));
    if (B->req_last) memcpy(B->req_last + om->req_offset, S.last, (size_t)n * sizeof(double));
  }
  if (om && om->decision_offset >= 0 && B->decisions) {
    int64_t c = S.dec_n < om->decision_capacity ? S.dec_n : om->decision_capacity;
    memcpy(B->decisions + om->decision_offset, S.dec, (size_t)c * sizeof(arrow_decision_t));
    if (S.dec_n > om->decision_capacity && sum->status == ARROW_OK) {
      sum->status = ARROW_BUFFER_OVERFLOW;
      sum->overflow = ARROW_OVF_DECISIONS;
    }
  }

  for (int i = 0; i < N; i++) inst_free(&S.inst[i]);
  free(S.inst); free(S.where);
  for (int k = 0; k < 4; k++) free(S.pool[k]);
  free(S.arrival); free(S.P); free(S.D); free(S.resident);
  free(S.first); free(S.last); free(S.ntok); free(tok_off);
  free(S.dec); free(S.heap.v);
  return sum->status;
}

typedef struct {
  const arrow_batch_t* B;
  atomic_int next;
  double* seconds;  /* optional: per-scenario wall seconds (bench.py's CPU baseline) */
} pool_job_t;

static double mono_now(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static void* pool_worker(void* arg) {
  pool_job_t* job = (pool_job_t*)arg;
  for (;;) {
    int k = atomic_fetch_add(&job->next, 1);
    if (k >= job->B->n_scenarios) break;
    int s = job->B->order ? job->B->order[k] : k;
    const double t0 = job->seconds ? mono_now() : 0.0;
    pdsim_oracle_run_one(job->B, s);
    if (job->seconds) job->seconds[s] = mono_now() - t0;
  }
  return NULL;
}

/* Scenarios are independent: a dynamic work queue over
 * n_threads POSIX threads, longest-first when the caller passes an order. */
int pdsim_oracle_run_batch(const arrow_batch_t* B, int n_threads) {
  return pdsim_oracle_run_batch_timed(B, n_threads, NULL);
}

int pdsim_oracle_run_batch_timed(const arrow_batch_t* B, int n_threads, double* seconds) {
  if (n_threads <= 0) n_threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (n_threads < 1) n_threads = 1;
  if (n_threads > B->n_scenarios) n_threads = B->n_scenarios > 0 ? B->n_scenarios : 1;
  pool_job_t job;
  job.B = B;
  job.seconds = seconds;
  atomic_init(&job.next, 0);
  if (n_threads == 1) {
    pool_worker(&job);
    return 1;
  }
  pthread_t* th = malloc((size_t)n_threads * sizeof(pthread_t));
  for (int t = 0; t < n_threads; t++) pthread_create(&th[t], NULL, pool_worker, &job);
  for (int t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
  free(th);
  return n_threads;
}
