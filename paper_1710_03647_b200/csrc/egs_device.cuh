// egs_device.cuh — value domain, cache-policy loads and warp/block primitives
// for the sm_100a energy-game kernels.
//
// Value domain (reference proj/include/egsolve/energy.hpp:14-31): a credit is
// a non-negative integer or top.  On the device the measure is held in the
// narrowest unsigned type that can represent every finite value <= credit_cap
// (u32 when credit_cap < 2^32 - 2, else u64) with top = all-ones, so that
// unsigned min/max order top above every finite credit exactly like the
// reference's INT64_MAX sentinel; the host widens top back to INT64_MAX.
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
// c_i > cap.  Finite f(t) <= cap < 2^63 - 2^31 and |w| < 2^31, so the int64
// difference never overflows.
template <class V>
__device__ __forceinline__ V ominus_cap(V ft, int32_t w, int64_t cap) {
  if (ft == Top<V>::v) return Top<V>::v;
  int64_t r = static_cast<int64_t>(ft) - static_cast<int64_t>(w);
  r = r < 0 ? 0 : r;
  return r > cap ? Top<V>::v : static_cast<V>(r);
}

// u32 path (cap < 2^32 - 1): the same value, written as selects so an
// unrolled row turns into straight-line predicated code.
template <>
__device__ __forceinline__ uint32_t ominus_cap<uint32_t>(uint32_t ft, int32_t w,
                                                         int64_t cap) {
  int64_t r = static_cast<int64_t>(ft) - static_cast<int64_t>(w);
  r = r < 0 ? 0 : r;
  uint32_t out = static_cast<uint32_t>(r);
  out = r > cap ? 0xFFFFFFFFu : out;
  return ft == 0xFFFFFFFFu ? 0xFFFFFFFFu : out;
}

// ------------------------------------------------------------ memory ----
// Mutable solver state (measure, witnesses, candidate flags, bitmaps) is
// read with ld.global.cg: it is written by other SMs inside the same
// persistent launch, so it must come from L2, never from a stale L1 line.
// The arena (offsets, edge records) is immutable during a solve: read-only
// path (ld.global.nc), edge records with the streaming hint so the
// once-per-round edge stream does not evict the L2-resident measure.
__device__ __forceinline__ uint32_t ldcg(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ uint64_t ldcg(const uint64_t* p) {
  return (uint64_t)__ldcg(reinterpret_cast<const unsigned long long*>(p));
}
__device__ __forceinline__ uint8_t ldcg(const uint8_t* p) {
  return (uint8_t)__ldcg(reinterpret_cast<const unsigned char*>(p));
}
__device__ __forceinline__ int2 ldcg(const int2* p) { return __ldcg(p); }
__device__ __forceinline__ void stcg(uint32_t* p, uint32_t v) { __stcg(p, v); }
__device__ __forceinline__ void stcg(uint64_t* p, uint64_t v) {
  __stcg(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}
__device__ __forceinline__ void stcg(uint8_t* p, uint8_t v) {
  __stcg(reinterpret_cast<unsigned char*>(p), (unsigned char)v);
}
__device__ __forceinline__ void stcg(int2* p, int2 v) { __stcg(p, v); }
__device__ __forceinline__ int2 ld_edge(const int2* p) { return __ldcs(p); }

// L2 eviction-priority policies (createpolicy; not volatile so the compiler
// hoists them).  The random gathers of the measure use evict_last so the
// measure stays L2-resident while the edge stream (evict_first) passes.
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint32_t gather(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(v)
               : "l"(p), "l"(l2_evict_last()));
  return v;
}
__device__ __forceinline__ uint64_t gather(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.cg.L2::cache_hint.u64 %0, [%1], %2;"
               : "=l"(v)
               : "l"(p), "l"(l2_evict_last()));
  return v;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ------------------------------------------------------ warp reduce ----
__device__ __forceinline__ uint32_t warp_min(uint32_t x) {
  return __reduce_min_sync(0xffffffffu, x);
}
__device__ __forceinline__ uint32_t warp_max(uint32_t x) {
  return __reduce_max_sync(0xffffffffu, x);
}
__device__ __forceinline__ uint64_t warp_min(uint64_t x) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const uint64_t y = __shfl_xor_sync(0xffffffffu, x, s);
    x = y < x ? y : x;
  }
  return x;
}
__device__ __forceinline__ uint64_t warp_max(uint64_t x) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const uint64_t y = __shfl_xor_sync(0xffffffffu, x, s);
    x = y > x ? y : x;
  }
  return x;
}
__device__ __forceinline__ unsigned long long warp_sum(unsigned long long x) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) x += __shfl_xor_sync(0xffffffffu, x, s);
  return x;
}

// Warp-aggregated append of `val` to list[*count++] for every lane with
// `pred`: one ballot, one atomicAdd per warp, popc ranks.  Warp-uniform call.
__device__ __forceinline__ void warp_append(bool pred, uint32_t val,
                                            uint32_t* list, uint32_t* count) {
  const uint32_t m = __ballot_sync(0xffffffffu, pred);
  if (m == 0u) return;
  const int leader = __ffs(m) - 1;
  uint32_t base = 0;
  if (lane_id() == (uint32_t)leader) base = atomicAdd(count, (uint32_t)__popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (pred) list[base + __popc(m & lanemask_lt())] = val;
}

// Warp-cooperative expansion of up to 32 index segments [b, e) (one per
// lane) into a flat stream: fn(item_index, owning_lane) is called once per
// item, 32 items per step, so one long segment (an R-MAT hub column) is
// shared by the whole warp instead of serialising one lane.  Warp-uniform.
// warp_expand with U items per lane per step (lane l takes items base + l,
// base + 32 + l, ...): fn(valid[U], idx[U]) can issue the loads of all U
// before it uses any.
template <int U, class Fn>
__device__ __forceinline__ void warp_expand_n(uint32_t b, uint32_t e, Fn&& fn) {
  const uint32_t lane = lane_id();
  const uint32_t len = e - b;
  uint32_t incl = len;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, s);
    if (lane >= (uint32_t)s) incl += y;
  }
  const uint32_t excl = incl - len;
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  for (uint32_t base = 0; base < total; base += 32 * U) {
    bool valid[U];
    uint32_t idx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t k = base + 32 * u + lane;
      uint32_t lo = 0;
#pragma unroll
      for (uint32_t step = 16; step > 0; step >>= 1) {
        const uint32_t c = lo + step;
        const uint32_t ex = __shfl_sync(0xffffffffu, excl, c & 31u);
        if (c < 32u && ex <= k) lo = c;
      }
      const uint32_t sb = __shfl_sync(0xffffffffu, b, lo);
      const uint32_t sx = __shfl_sync(0xffffffffu, excl, lo);
      valid[u] = k < total;
      idx[u] = sb + (k - sx);
    }
    fn(valid, idx);
  }
}

template <class Fn>
__device__ __forceinline__ void warp_expand(uint32_t b, uint32_t e, Fn&& fn) {
  const uint32_t lane = lane_id();
  const uint32_t len = e - b;
  uint32_t incl = len;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, s);
    if (lane >= (uint32_t)s) incl += y;
  }
  const uint32_t excl = incl - len;
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  for (uint32_t base = 0; base < total; base += 32) {
    const uint32_t k = base + lane;
    // last lane s with excl[s] <= k (excl is non-decreasing)
    uint32_t lo = 0;
#pragma unroll
    for (uint32_t step = 16; step > 0; step >>= 1) {
      const uint32_t c = lo + step;
      const uint32_t ex = __shfl_sync(0xffffffffu, excl, c & 31u);
      if (c < 32u && ex <= k) lo = c;
    }
    const uint32_t sb = __shfl_sync(0xffffffffu, b, lo);
    const uint32_t sx = __shfl_sync(0xffffffffu, excl, lo);
    fn(k < total, sb + (k - sx), lo);
  }
}

// ------------------------------------------------ TMA bulk copies ----
// 1-D bulk copies global -> shared (cp.async.bulk, SASS UBLKCP) completing
// on an mbarrier transaction count.  Source/destination 16-byte aligned,
// size a multiple of 16.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
// make barrier initialisation visible to the async (TMA) proxy
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// order earlier generic-proxy accesses of a buffer before an async-proxy
// write into it (buffer reuse)
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(l2_evict_first())
      : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// A transfer that never lands (a bug, or a faulted copy) traps instead of
// hanging the persistent grid (~2^22 polls, far beyond any copy latency).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t spins = 0;
  while (!mbar_try_wait(bar, parity)) {
    if (++spins > (1u << 22)) __trap();
  }
}

}  // namespace egs
