// emu.cpp — TEST-ONLY host emulation of one warp per scenario.
//
// Each lane is a host thread running the very same Sim<> code the CUDA
// kernel runs (csrc/sim_core.cuh); warp collectives become barrier-
// synchronised exchanges through a shared slot array.  This lets the
// kernel's scheduling logic be debugged against the CPU oracle in a
// container without a GPU.  It is never loaded by the product path
// (paper_2505_11916_b200 only loads the CUDA library).
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "../sim_core.cuh"

namespace {

struct SpinBarrier {
  std::atomic<int> count{0};
  std::atomic<int> phase{0};
  int n = 1;
  void wait() {
    int ph = phase.load(std::memory_order_acquire);
    if (count.fetch_add(1, std::memory_order_acq_rel) + 1 == n) {
      count.store(0, std::memory_order_relaxed);
      phase.fetch_add(1, std::memory_order_acq_rel);
      return;
    }
    int spins = 0;
    while (phase.load(std::memory_order_acquire) == ph) {
      if (++spins > 64) {
        std::this_thread::yield();
        spins = 0;
      }
    }
  }
};

template <int WIDTH_>
struct EmuWarp {
  static constexpr int WIDTH = WIDTH_;
  struct Shared {
    SpinBarrier bar;
    uint64_t slot[WIDTH_];
  };
  Shared* sh;
  int ln;

  int lane() const { return ln; }
  void sync() const { sh->bar.wait(); }

  uint64_t get(uint64_t v, int src) const {
    sh->slot[ln] = v;
    sync();
    uint64_t r = sh->slot[src];
    sync();
    return r;
  }
  template <class F>
  uint64_t fold(uint64_t v, F f) const {
    sh->slot[ln] = v;
    sync();
    uint64_t r = sh->slot[0];
    for (int i = 1; i < WIDTH; i++) r = f(r, sh->slot[i]);
    sync();
    return r;
  }
  uint32_t ballot(bool p) const {
    return (uint32_t)fold(p ? 1ull << ln : 0ull, [](uint64_t a, uint64_t b) { return a | b; });
  }
  bool any(bool p) const { return ballot(p) != 0; }
  uint32_t shfl(uint32_t v, int src) const { return (uint32_t)get(v, src); }
  int32_t shfl(int32_t v, int src) const { return (int32_t)(uint32_t)get((uint32_t)v, src); }
  uint64_t shfl(uint64_t v, int src) const { return get(v, src); }
  int64_t shfl(int64_t v, int src) const { return (int64_t)get((uint64_t)v, src); }
  double shfl(double v, int src) const {
    uint64_t u;
    memcpy(&u, &v, 8);
    u = get(u, src);
    double r;
    memcpy(&r, &u, 8);
    return r;
  }
  uint32_t min_u32(uint32_t v) const {
    return (uint32_t)fold(v, [](uint64_t a, uint64_t b) { return a < b ? a : b; });
  }
  uint32_t max_u32(uint32_t v) const {
    return (uint32_t)fold(v, [](uint64_t a, uint64_t b) { return a > b ? a : b; });
  }
  uint32_t add_u32(uint32_t v) const {
    return (uint32_t)fold(v, [](uint64_t a, uint64_t b) { return (uint64_t)(uint32_t)(a + b); });
  }
  uint32_t match_any(uint64_t v) const {
    sh->slot[ln] = v;
    sync();
    uint32_t m = 0;
    for (int i = 0; i < WIDTH; i++)
      if (sh->slot[i] == v) m |= 1u << i;
    sync();
    return m;
  }
  uint32_t match_any_u32(uint32_t v) const { return match_any((uint64_t)v); }
  int atomic_add_shared(int* p, int v) const { return __atomic_fetch_add(p, v, __ATOMIC_RELAXED); }
};

template <int W, int IPL>
void run_scenario(const arrow_batch_t* b, int s, const arrow::SlotLayout& L, char* ws) {
  using Warp = EmuWarp<W>;
  typename Warp::Shared shared;
  shared.bar.n = W;
  arrow::WarpSmem* sm = (arrow::WarpSmem*)calloc(1, sizeof(arrow::WarpSmem));
  std::vector<std::thread> th;
  for (int ln = 0; ln < W; ln++) {
    th.emplace_back([&, ln] {
      arrow::Sim<Warp, IPL> sim;
      sim.w.sh = &shared;
      sim.w.ln = ln;
      sim.lane = ln;
      sim.sm = sm;
      sim.B = b;
      sim.L = L;
      sim.p = arrow::slot_ptrs(ws, L);
      sim.run(s);
    });
  }
  for (auto& t : th) t.join();
  free(sm);
}

template <int W>
int run_width(const arrow_batch_t* b) {
  arrow::SlotLayout L = arrow::make_layout(b->max_requests, b->max_instances, b->queue_capacity,
                                           b->running_capacity, b->emission_capacity);
  char* ws = (char*)aligned_alloc(256, (size_t)L.bytes);
  if (!ws) return -1;
  int ipl = (b->max_instances + W - 1) / W;
  for (int k = 0; k < b->n_scenarios; k++) {
    int s = b->order ? b->order[k] : k;
    if (ipl <= 1)
      run_scenario<W, 1>(b, s, L, ws);
    else
      run_scenario<W, 2>(b, s, L, ws);
  }
  free(ws);
  return 0;
}

}  // namespace

extern "C" int arrow_emu_run(const arrow_batch_t* b, int width) {
  if (width == 4) {
    if (b->max_instances > 8) return -2;
    return run_width<4>(b);
  }
  if (width == 8) {
    if (b->max_instances > 16) return -2;
    return run_width<8>(b);
  }
  if (width == 32) {
    if (b->max_instances > 64) return -2;
    return run_width<32>(b);
  }
  return -3;
}
