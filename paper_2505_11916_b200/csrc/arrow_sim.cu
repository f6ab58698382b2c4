// arrow_sim.cu — sm_100a persistent kernel + C-ABI (include/arrow_sim.h).
//
// One warp = one scenario slot.  The grid is sized to the device's resident
// warp capacity (SM count x blocks/SM from the occupancy API); warps pull
// scenario ids from an atomic counter, so long scenarios (10^5-10^6 events)
// and short ones (10^3) balance dynamically.  Each slot owns a private
// region of the caller's workspace (queues, rings, per-request state) sized
// by make_layout(); traces are shared read-only by every slot.
#include <cuda_runtime.h>
#include <stddef.h>

#include "arrow_sim.h"
#include "sim_core.cuh"

namespace {

#ifndef ARROW_LAT_WARPS
#define ARROW_LAT_WARPS 2
#endif
#ifndef ARROW_TP_WARPS
#define ARROW_TP_WARPS 4
#endif
constexpr int kWarpsPerBlock = ARROW_TP_WARPS;
constexpr int kThreads = kWarpsPerBlock * 32;
// Two builds of the kernel: MINB = 1 lets the compiler use every register it
// wants (shortest per-scenario chains: a sweep that fits in one wave of
// resident warps finishes when its longest scenario does); MINB = 3 caps
// registers at 168 so three blocks (12 warps) share an SM (throughput for
// sweeps of many waves, where issue slots, not chain latency, are the bound).
#ifndef ARROW_TP_BLOCKS
#define ARROW_TP_BLOCKS 3
#endif
constexpr int kMinBlocksThroughput = ARROW_TP_BLOCKS;
// two instances per lane (N > 32) carry twice the register state
#ifndef ARROW_TP_BLOCKS_IPL2
#define ARROW_TP_BLOCKS_IPL2 3
#endif
constexpr int kMinBlocksThroughput2 = ARROW_TP_BLOCKS_IPL2;
constexpr int kLatWarps = ARROW_LAT_WARPS;  // warps per block of the latency build

// LEAN: summaries-only batches (no outmap): every optional-output write
// compiles out of the event loop (smaller hot code; the occupancy build is
// instruction-fetch bound).  The audit build keeps one variant.
#ifdef ARROW_AUDIT
constexpr bool kLeanBuild = false;
#else
constexpr bool kLeanBuild = true;
#endif

template <int IPL, int MINB, int WPB, bool LEAN>
__global__ void __launch_bounds__(WPB * 32, MINB) arrow_sim_kernel(const arrow_batch_t batch, char* workspace,
                                                                   arrow::SlotLayout L, int* counter, int n_slots) {
  __shared__ arrow::WarpSmem smem[WPB];
  __shared__ arrow_batch_t sb;
  if (threadIdx.x == 0) sb = batch;
  __syncthreads();
  const int wid = threadIdx.x >> 5;
  const int slot = blockIdx.x * WPB + wid;
  if (slot >= n_slots) return;
  arrow::Sim<DevWarp, IPL, (MINB > 1), LEAN> sim;   // occupancy build: COMPACT code
  sim.sm = &smem[wid];
  sim.B = &sb;
  sim.L = L;
  sim.p = arrow::slot_ptrs(workspace + (int64_t)slot * L.bytes, L);
  sim.lane = (int)(threadIdx.x & 31u);
  for (;;) {
    int k = 0;
    if (sim.lane == 0) k = atomicAdd(counter, 1);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= sb.n_scenarios) break;
    const int s = sb.order ? sb.order[k] : k;
    sim.run(s);
  }
}

arrow::SlotLayout layout_of(const arrow_batch_t* b) {
  return arrow::make_layout(b->max_requests, b->max_instances, b->queue_capacity, b->running_capacity,
                            b->emission_capacity);
}

int ipl_of(const arrow_batch_t* b) { return b->max_instances > 32 ? 2 : 1; }

template <int IPL, int MINB, int WPB>
cudaError_t capacity_of(int sms, long long* cap) {
  int per_sm = 0;
  cudaError_t e =
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, arrow_sim_kernel<IPL, MINB, WPB, false>, WPB * 32, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  *cap = (long long)sms * per_sm * WPB;
  return cudaSuccess;
}

// Resident scenario slots and the kernel build: the latency build when the
// whole batch fits in its single wave, the occupancy build otherwise.
cudaError_t slots_for(const arrow_batch_t* b, int* slots, bool* throughput) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  int sms = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  long long lat = 0, thr = 0;
  if (ipl_of(b) == 2) {
    if ((e = capacity_of<2, 1, kLatWarps>(sms, &lat)) != cudaSuccess) return e;
    if ((e = capacity_of<2, kMinBlocksThroughput2, kWarpsPerBlock>(sms, &thr)) != cudaSuccess) return e;
  } else {
    if ((e = capacity_of<1, 1, kLatWarps>(sms, &lat)) != cudaSuccess) return e;
    if ((e = capacity_of<1, kMinBlocksThroughput, kWarpsPerBlock>(sms, &thr)) != cudaSuccess) return e;
  }
  const long long want = b->n_scenarios > 0 ? b->n_scenarios : 1;
  bool tp = want > lat;
  if (b->flags & ARROW_SIM_FORCE_LATENCY) tp = false;
  if (b->flags & ARROW_SIM_FORCE_THROUGHPUT) tp = true;
  const long long cap = tp ? thr : lat;
  *slots = (int)(want < cap ? want : cap);
  if (throughput) *throughput = tp;
  return cudaSuccess;
}

}  // namespace

extern "C" {

int arrow_sim_abi_version(void) { return ARROW_SIM_ABI_VERSION; }

int arrow_sim_slots(const arrow_batch_t* b, int* slots) { return (int)slots_for(b, slots, nullptr); }

int arrow_sim_workspace_size(const arrow_batch_t* b, size_t* bytes) {
  if (!b || !bytes) return (int)cudaErrorInvalidValue;
  if (b->max_instances < 1 || b->max_instances > arrow::MAX_INST) return (int)cudaErrorInvalidValue;
  int slots = 0;
  cudaError_t e = slots_for(b, &slots, nullptr);
  if (e != cudaSuccess) return (int)e;
  arrow::SlotLayout L = layout_of(b);
  *bytes = (size_t)slots * (size_t)L.bytes + 256;
  return 0;
}

int arrow_sim_run(const arrow_batch_t* b, void* workspace, size_t workspace_bytes, void* stream) {
  if (!b) return (int)cudaErrorInvalidValue;
  if (b->n_scenarios <= 0) return 0;
  size_t need = 0;
  int rc = arrow_sim_workspace_size(b, &need);
  if (rc) return rc;
  if (!workspace || workspace_bytes < need) return (int)cudaErrorInvalidValue;
  int slots = 0;
  bool tp = false;
  cudaError_t e = slots_for(b, &slots, &tp);
  if (e != cudaSuccess) return (int)e;
  arrow::SlotLayout L = layout_of(b);
  char* ws = (char*)workspace;
  int* counter = (int*)(ws + (size_t)slots * (size_t)L.bytes);
  cudaStream_t st = (cudaStream_t)stream;
  e = cudaMemsetAsync(counter, 0, sizeof(int), st);
  if (e != cudaSuccess) return (int)e;
  const int wpb = tp ? kWarpsPerBlock : kLatWarps;
  const int grid = (slots + wpb - 1) / wpb;
  const bool lean = kLeanBuild && b->outmap == nullptr;
#define ARROW_LAUNCH(IPL_, MINB_, WPB_)                                                                  \
  do {                                                                                                  \
    if (lean)                                                                                           \
      arrow_sim_kernel<IPL_, MINB_, WPB_, kLeanBuild><<<grid, (WPB_) * 32, 0, st>>>(*b, ws, L, counter, slots); \
    else                                                                                                \
      arrow_sim_kernel<IPL_, MINB_, WPB_, false><<<grid, (WPB_) * 32, 0, st>>>(*b, ws, L, counter, slots);     \
  } while (0)
  if (ipl_of(b) == 2) {
    if (tp)
      ARROW_LAUNCH(2, kMinBlocksThroughput2, kWarpsPerBlock);
    else
      ARROW_LAUNCH(2, 1, kLatWarps);
  } else {
    if (tp)
      ARROW_LAUNCH(1, kMinBlocksThroughput, kWarpsPerBlock);
    else
      ARROW_LAUNCH(1, 1, kLatWarps);
  }
#undef ARROW_LAUNCH
  return (int)cudaGetLastError();
}

// Struct sizes followed by every field offset, in declaration order, so host
// bindings can verify their mirrors (tests/test_abi.py).  No CUDA calls.
#define OFF(T, f) (int64_t) offsetof(T, f)
int arrow_sim_layout(int64_t* out, int cap) {
  const int64_t v[] = {
    (int64_t)sizeof(arrow_scenario_t), (int64_t)sizeof(arrow_outmap_t), (int64_t)sizeof(arrow_summary_t),
    (int64_t)sizeof(arrow_decision_t), (int64_t)sizeof(arrow_snapshot_t), (int64_t)sizeof(arrow_instdiag_t),
    (int64_t)sizeof(arrow_batch_t),
    OFF(arrow_scenario_t, trace_offset),
    OFF(arrow_scenario_t, n_requests),
    OFF(arrow_scenario_t, n_instances),
    OFF(arrow_scenario_t, n_prefill_init),
    OFF(arrow_scenario_t, strategy),
    OFF(arrow_scenario_t, enable_flips),
    OFF(arrow_scenario_t, kv_capacity),
    OFF(arrow_scenario_t, chunk_budget),
    OFF(arrow_scenario_t, max_batch),
    OFF(arrow_scenario_t, bytes_per_token),
    OFF(arrow_scenario_t, max_tokens),
    OFF(arrow_scenario_t, stall_limit),
    OFF(arrow_scenario_t, arrival_scale),
    OFF(arrow_scenario_t, true_a2),
    OFF(arrow_scenario_t, true_a1),
    OFF(arrow_scenario_t, true_a0),
    OFF(arrow_scenario_t, pred_a2),
    OFF(arrow_scenario_t, pred_a1),
    OFF(arrow_scenario_t, pred_a0),
    OFF(arrow_scenario_t, b1),
    OFF(arrow_scenario_t, b0),
    OFF(arrow_scenario_t, base_latency),
    OFF(arrow_scenario_t, bandwidth),
    OFF(arrow_scenario_t, ttft_slo),
    OFF(arrow_scenario_t, tpot_slo),
    OFF(arrow_scenario_t, ttft_thr),
    OFF(arrow_scenario_t, tpot_thr),
    OFF(arrow_scenario_t, theta_d),
    OFF(arrow_scenario_t, theta_busy),
    OFF(arrow_scenario_t, breach_duration),
    OFF(arrow_scenario_t, monitor_period),
    OFF(arrow_scenario_t, window),
    OFF(arrow_scenario_t, min_iteration),
    OFF(arrow_outmap_t, req_offset),
    OFF(arrow_outmap_t, decision_offset),
    OFF(arrow_outmap_t, decision_capacity),
    OFF(arrow_outmap_t, snapshot_offset),
    OFF(arrow_outmap_t, snapshot_capacity),
    OFF(arrow_outmap_t, iterlog_offset),
    OFF(arrow_outmap_t, iterlog_stride),
    OFF(arrow_outmap_t, diag_offset),
    OFF(arrow_outmap_t, token_offset),
    OFF(arrow_summary_t, status),
    OFF(arrow_summary_t, overflow),
    OFF(arrow_summary_t, n_requests),
    OFF(arrow_summary_t, n_completed),
    OFF(arrow_summary_t, n_ok),
    OFF(arrow_summary_t, n_flips),
    OFF(arrow_summary_t, n_events),
    OFF(arrow_summary_t, n_iterations),
    OFF(arrow_summary_t, n_decisions),
    OFF(arrow_summary_t, n_ticks),
    OFF(arrow_summary_t, n_snapshots),
    OFF(arrow_summary_t, stall_time),
    OFF(arrow_summary_t, attainment),
    OFF(arrow_summary_t, p90_ttft),
    OFF(arrow_summary_t, p90_tpot),
    OFF(arrow_summary_t, mean_ttft),
    OFF(arrow_summary_t, mean_tpot),
    OFF(arrow_summary_t, goodput),
    OFF(arrow_summary_t, span),
    OFF(arrow_summary_t, decision_hash),
    OFF(arrow_summary_t, n_serial_steps),
    OFF(arrow_summary_t, n_parallel_steps),
    OFF(arrow_summary_t, cycles),
    OFF(arrow_summary_t, reserved),
    OFF(arrow_decision_t, time),
    OFF(arrow_decision_t, request),
    OFF(arrow_decision_t, instance),
    OFF(arrow_decision_t, kind),
    OFF(arrow_decision_t, code),
    OFF(arrow_snapshot_t, time),
    OFF(arrow_snapshot_t, pred_delay),
    OFF(arrow_snapshot_t, avg_interval),
    OFF(arrow_snapshot_t, instance),
    OFF(arrow_snapshot_t, pool),
    OFF(arrow_snapshot_t, running_tokens),
    OFF(arrow_snapshot_t, kv_used),
    OFF(arrow_snapshot_t, queue_len),
    OFF(arrow_snapshot_t, prefill_count),
    OFF(arrow_snapshot_t, decode_count),
    OFF(arrow_snapshot_t, reserved),
    OFF(arrow_instdiag_t, busy_until),
    OFF(arrow_instdiag_t, pool),
    OFF(arrow_instdiag_t, kv_used),
    OFF(arrow_instdiag_t, running),
    OFF(arrow_instdiag_t, waiting),
    OFF(arrow_instdiag_t, migrating),
    OFF(arrow_instdiag_t, reserved),
    OFF(arrow_batch_t, n_scenarios),
    OFF(arrow_batch_t, flags),
    OFF(arrow_batch_t, max_requests),
    OFF(arrow_batch_t, max_instances),
    OFF(arrow_batch_t, queue_capacity),
    OFF(arrow_batch_t, emission_capacity),
    OFF(arrow_batch_t, running_capacity),
    OFF(arrow_batch_t, fifo_capacity),
    OFF(arrow_batch_t, arrival),
    OFF(arrow_batch_t, input_len),
    OFF(arrow_batch_t, output_len),
    OFF(arrow_batch_t, scenarios),
    OFF(arrow_batch_t, order),
    OFF(arrow_batch_t, outmap),
    OFF(arrow_batch_t, summaries),
    OFF(arrow_batch_t, req_first),
    OFF(arrow_batch_t, req_last),
    OFF(arrow_batch_t, req_prefill),
    OFF(arrow_batch_t, req_decode),
    OFF(arrow_batch_t, req_decode_iter),
    OFF(arrow_batch_t, decisions),
    OFF(arrow_batch_t, snapshots),
    OFF(arrow_batch_t, iterlog),
    OFF(arrow_batch_t, diag),
    OFF(arrow_batch_t, token_times),
  };
  const int n = (int)(sizeof(v) / sizeof(v[0]));
  for (int i = 0; i < n && i < cap; i++) out[i] = v[i];
  return n;
}
#undef OFF

const char* arrow_sim_status_string(int status) {
  switch (status) {
    case ARROW_OK: return "ok";
    case ARROW_STALLED: return "stalled";
    case ARROW_INCOMPLETE: return "incomplete";
    case ARROW_NOT_DRAINED: return "not-drained";
    case ARROW_NO_INSTANCE: return "no-instance";
    case ARROW_ZERO_DIVISION: return "zero-division";
    case ARROW_BUFFER_OVERFLOW: return "buffer-overflow";
    case ARROW_INTERNAL: return "internal";
    case ARROW_AUDIT_FAILED: return "audit-failed";
    default: return "unknown";
  }
}

}  // extern "C"

#ifdef ARROW_PROF
// Profiling build only (-DARROW_PROF): serial-step cycles by event kind per
// scenario id (arrival, -, prefill-complete, -, tick, loud iteration,
// migration, rescan), copied out after a launch.
extern "C" int arrow_sim_prof(int64_t* out, int n) {
  if (n > ARROW_PROF_MAX) n = ARROW_PROF_MAX;
  return (int)cudaMemcpyFromSymbol(out, arrow_prof_cycles, (size_t)n * 32 * sizeof(int64_t));
}
#endif
