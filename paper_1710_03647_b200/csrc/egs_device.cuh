// egs_device.cuh — value domain and warp/group primitives for the sm_100a
// energy-game kernels.
//
// Value domain (reference proj/include/egsolve/energy.hpp:14-31): a credit is
// a non-negative integer or top.  On the device the measure is held in the
// narrowest unsigned type that can represent every finite value <= credit_cap
// (u32 when credit_cap < 2^32 - 1, else u64) with top = all-ones; the host
// widens top back to INT64_MAX on copy-out.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace egs {

template <class V>
struct Top;
template <>
struct Top<uint32_t> {
  static constexpr uint32_t v = 0xFFFFFFFFu;
};
template <>
struct Top<uint64_t> {
  static constexpr uint64_t v = 0xFFFFFFFFFFFFFFFFull;
};

// f(t) ⊖ w saturated against the credit bound: raw_ominus (energy.hpp:20-31)
// followed by the lift's `acc > credit_cap ? top : acc` (measure_ops.hpp:51).
// Applying the cap per candidate is value-identical to applying it to the
// min/max: min(c_i) > cap iff every c_i > cap; max(c_i) > cap iff some
// c_i > cap.  Finite f(t) <= cap and |w| < 2^31, so the int64 difference
// never overflows.
template <class V>
__device__ __forceinline__ V ominus_cap(V ft, int32_t w, int64_t cap) {
  if (ft == Top<V>::v) return Top<V>::v;
  int64_t r = static_cast<int64_t>(ft) - static_cast<int64_t>(w);
  r = r < 0 ? 0 : r;
  return r > cap ? Top<V>::v : static_cast<V>(r);
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Min (player 0) or max (player 1) across the G aligned lanes of a group.
// Every lane of the warp must call it (full-mask shuffles).
template <int G, class T>
__device__ __forceinline__ T group_minmax(T x, bool is_min) {
#pragma unroll
  for (int s = G / 2; s > 0; s >>= 1) {
    T y = __shfl_xor_sync(0xffffffffu, x, s);
    x = is_min ? (y < x ? y : x) : (y > x ? y : x);
  }
  return x;
}

template <int G>
__device__ __forceinline__ uint32_t group_mask() {
  if constexpr (G == 32) {
    return 0xffffffffu;
  } else {
    return ((1u << G) - 1u) << (lane_id() & ~(uint32_t)(G - 1));
  }
}

template <int G>
__device__ __forceinline__ bool group_any(bool p) {
  return (__ballot_sync(0xffffffffu, p) & group_mask<G>()) != 0u;
}

template <int G>
__device__ __forceinline__ bool group_all(bool p) {
  return (__ballot_sync(0xffffffffu, p) & group_mask<G>()) == group_mask<G>();
}

// Warp-aggregated append of `val` to list[*count++] for every lane with
// `pred`: one ballot, one atomicAdd per converged subset, popc ranks.
__device__ __forceinline__ void warp_append(bool pred, uint32_t val,
                                            uint32_t* list, uint32_t* count) {
  const uint32_t act = __activemask();
  const uint32_t m = __ballot_sync(act, pred);
  if (m == 0u) return;
  const uint32_t lane = lane_id();
  const int leader = __ffs(m) - 1;
  uint32_t base = 0;
  if (lane == (uint32_t)leader) base = atomicAdd(count, (uint32_t)__popc(m));
  base = __shfl_sync(act, base, leader);
  if (pred) list[base + __popc(m & ((1u << lane) - 1u))] = val;
}

// Sum a per-thread counter over the warp and add it once to *dst.
// Must be called by all 32 lanes.
__device__ __forceinline__ void warp_add_u64(unsigned long long x,
                                             unsigned long long* dst) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) x += __shfl_xor_sync(0xffffffffu, x, s);
  if (lane_id() == 0 && x != 0ull) atomicAdd(dst, x);
}

}  // namespace egs
