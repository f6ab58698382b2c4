// warp.cuh — the warp-collective primitives the scenario simulator is written
// against.  DevWarp maps them onto sm_100a warp intrinsics (shfl / vote /
// redux.sync).  The same simulator source is also instantiated on the host
// with a thread-per-lane emulation (tests only, csrc/emu/), which is how its
// logic is checked against the CPU oracle without a GPU.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define AS_HD __host__ __device__ __forceinline__
#define AS_DEV __device__ __forceinline__
#else
#define AS_HD inline
#define AS_DEV inline
#endif

#ifdef __CUDACC__
struct DevWarp {
  static constexpr int WIDTH = 32;
  static constexpr uint32_t FULL = 0xffffffffu;
  AS_DEV int lane() const { return (int)(threadIdx.x & 31u); }
  AS_DEV void sync() const { __syncwarp(FULL); }
  AS_DEV uint32_t ballot(bool p) const { return __ballot_sync(FULL, p); }
  AS_DEV bool any(bool p) const { return __any_sync(FULL, p) != 0; }
  AS_DEV uint32_t shfl(uint32_t v, int src) const { return __shfl_sync(FULL, v, src); }
  AS_DEV int32_t shfl(int32_t v, int src) const { return __shfl_sync(FULL, v, src); }
  AS_DEV uint64_t shfl(uint64_t v, int src) const { return __shfl_sync(FULL, v, src); }
  AS_DEV int64_t shfl(int64_t v, int src) const { return __shfl_sync(FULL, v, src); }
  AS_DEV double shfl(double v, int src) const { return __shfl_sync(FULL, v, src); }
  AS_DEV uint32_t min_u32(uint32_t v) const { return __reduce_min_sync(FULL, v); }
  AS_DEV uint32_t max_u32(uint32_t v) const { return __reduce_max_sync(FULL, v); }
  AS_DEV uint32_t add_u32(uint32_t v) const { return __reduce_add_sync(FULL, v); }
  AS_DEV uint32_t match_any(uint64_t v) const { return __match_any_sync(FULL, v); }
  AS_DEV uint32_t match_any_u32(uint32_t v) const { return __match_any_sync(FULL, v); }
  AS_DEV int atomic_add_shared(int* p, int v) const { return atomicAdd(p, v); }
};
#endif
