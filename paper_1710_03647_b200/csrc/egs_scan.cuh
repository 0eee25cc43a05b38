// egs_scan.cuh — hand-written device primitives of the arena build
// (egs_build.cuh / egs_solver.cu), replacing library scans and sorts:
//
//   * exclusive prefix sum of u32 / u64 arrays (reduce -> scan of the tile
//     sums -> down-sweep), in place allowed;
//   * the stable class placement of the relabelling: every vertex's
//     position in the class-sorted order (player 0 light / medium / heavy,
//     player 1 light / medium / heavy; reorder_by_owner arena.cpp:119-149
//     refined by degree) from per-tile class counts and warp ballots --
//     a stable 6-bucket counting sort, mapped through the multi-GPU plan.
#pragma once

#include <cstdint>

#include "egs_device.cuh"
#include "egs_types.cuh"

namespace egs {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;  // per thread: tiles of 4096 elements
constexpr uint32_t kScanTile = kScanThreads * kScanItems;

// block-wide exclusive scan of one value per thread; *total = block sum
template <class T>
__device__ __forceinline__ T block_excl_scan(T x, T* s_warp, T* total) {
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  T incl = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= (uint32_t)d) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    T w = lane < (uint32_t)(blockDim.x >> 5) ? s_warp[lane] : T(0);
    T wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= (uint32_t)d) wi += y;
    }
    if (lane < (uint32_t)(blockDim.x >> 5)) s_warp[lane] = wi - w;
    if (lane == 31) s_warp[32] = wi;
  }
  __syncthreads();
  const T out = s_warp[warp] + incl - x;
  if (total) *total = s_warp[32];
  __syncthreads();
  return out;
}

// tile sums: tsum[t] = sum of in[t * kScanTile ...] (grid-stride over tiles)
template <class T, class In>
__global__ void __launch_bounds__(kScanThreads)
    k_scan_reduce(const In* in, uint64_t n, T* tsum, uint64_t ntiles) {
  __shared__ T s_warp[33];
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t base = t * kScanTile;
    T acc = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const uint64_t i = base + (uint64_t)k * kScanThreads + threadIdx.x;
      if (i < n) acc += (T)in[i];
    }
    T total;
    block_excl_scan<T>(acc, s_warp, &total);
    if (threadIdx.x == 0) tsum[t] = total;
  }
}

// exclusive scan of the tile sums in place (one CTA, sequential chunks)
template <class T>
__global__ void __launch_bounds__(1024) k_scan_tiles(T* tsum, uint64_t ntiles) {
  __shared__ T s_warp[33];
  T carry = 0;
  for (uint64_t base = 0; base < ntiles; base += blockDim.x) {
    const uint64_t i = base + threadIdx.x;
    const T x = i < ntiles ? tsum[i] : T(0);
    T total;
    const T ex = block_excl_scan<T>(x, s_warp, &total);
    if (i < ntiles) tsum[i] = carry + ex;
    carry += total;
  }
}

// out[i] = tsum[tile] + exclusive scan of the tile's in[] (blocked per
// thread so the scan is over consecutive elements)
template <class T, class In>
__global__ void __launch_bounds__(kScanThreads)
    k_scan_down(const In* in, T* out, uint64_t n, const T* tsum, uint64_t ntiles) {
  __shared__ T s_warp[33];
  __shared__ T s_buf[kScanTile];
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t base = t * kScanTile;
    // coalesced load into shared memory, then each thread scans its run
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const uint64_t i = base + (uint64_t)k * kScanThreads + threadIdx.x;
      s_buf[k * kScanThreads + threadIdx.x] = i < n ? (T)in[i] : T(0);
    }
    __syncthreads();
    T run[kScanItems];
    T acc = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      run[k] = acc;
      acc += s_buf[threadIdx.x * kScanItems + k];
    }
    const T off = tsum[t] + block_excl_scan<T>(acc, s_warp, nullptr);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) s_buf[threadIdx.x * kScanItems + k] = off + run[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const uint64_t i = base + (uint64_t)k * kScanThreads + threadIdx.x;
      if (i < n) out[i] = s_buf[k * kScanThreads + threadIdx.x];
    }
    __syncthreads();
  }
}

// ------------------------------------------------- class placement ----
// Class of every vertex (key[v]) and per-tile class counts, class-major:
// tcount[c * ntiles + tile].
__global__ void __launch_bounds__(kScanThreads)
    k_class_tiles(uint32_t n, const uint64_t* off64, const uint8_t* owner, uint8_t* key,
                  uint32_t* tcount, uint32_t ntiles, unsigned int* hist) {
  __shared__ unsigned int s_cnt[kNumClasses];
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (threadIdx.x < kNumClasses) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    unsigned int mine[kNumClasses] = {0, 0, 0, 0, 0, 0};
    for (int k = 0; k < kScanItems; ++k) {
      const uint32_t v = t * kScanTile + k * kScanThreads + threadIdx.x;
      if (v < n) {
        const uint64_t deg = off64[v + 1] - off64[v];
        const int c = (owner[v] ? 3 : 0) + (deg <= kLightMax ? 0 : deg <= kMediumMax ? 1 : 2);
        key[v] = (uint8_t)c;
#pragma unroll
        for (int cc = 0; cc < kNumClasses; ++cc) mine[cc] += c == cc;
      }
    }
#pragma unroll
    for (int cc = 0; cc < kNumClasses; ++cc) {
      const unsigned int w = __reduce_add_sync(0xffffffffu, mine[cc]);
      if (lane_id() == 0 && w) atomicAdd(&s_cnt[cc], w);
    }
    __syncthreads();
    if (threadIdx.x < kNumClasses) {
      tcount[threadIdx.x * ntiles + t] = s_cnt[threadIdx.x];
      if (s_cnt[threadIdx.x]) atomicAdd(hist + threadIdx.x, s_cnt[threadIdx.x]);
    }
    __syncthreads();
  }
}

// The partition of the class-sorted order (egs_part_plan, include/egs_gpu.h)
// as the build kernels need it: class k's piece r covers class positions
// [piece[k][r], piece[k][r+1]) and is relabelled from id cls_lo[r][k] on.
struct PlanDev {
  uint32_t world;
  uint32_t piece[kNumClasses][kMaxRanks + 1];
  uint32_t cls_lo[kMaxRanks][kNumClasses + 1];
};

// new id of the vertex at position `pos` of class c (0-based in the class);
// one rank: the class-sorted position itself (cls_lo unused)
__device__ __forceinline__ uint32_t plan_new_id(const PlanDev& pl, int c, uint32_t pos) {
  uint32_t r = 0;
  while (r + 1 < pl.world && pos >= pl.piece[c][r + 1]) ++r;
  return pl.cls_lo[r][c] + (pos - pl.piece[c][r]);
}

// Stable placement: position of v in its class = tpos[c * ntiles + tile]
// (exclusive scan of tcount, minus the class start) + the count of class-c
// vertices before v in the tile (steps of 256 in order, warp ballots, warp
// prefixes); perm[v] = new id, inv[new id] = v.
__global__ void __launch_bounds__(kScanThreads)
    k_class_place(uint32_t n, const uint8_t* key, const uint32_t* tpos, uint32_t ntiles,
                  const __grid_constant__ PlanDev pl, uint32_t* perm, uint32_t* inv) {
  constexpr int W = kScanThreads / 32;
  __shared__ uint32_t s_wc[W][kNumClasses];
  __shared__ uint32_t s_run[kNumClasses];
  __shared__ uint32_t s_cstart[kNumClasses];
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  if (threadIdx.x < kNumClasses) s_cstart[threadIdx.x] = tpos[threadIdx.x * ntiles];
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (threadIdx.x < kNumClasses) s_run[threadIdx.x] = tpos[threadIdx.x * ntiles + t];
    __syncthreads();
    for (int k = 0; k < kScanItems; ++k) {
      const uint32_t v = t * kScanTile + k * kScanThreads + threadIdx.x;
      const int c = v < n ? key[v] : -1;
      uint32_t rank = 0;
#pragma unroll
      for (int cc = 0; cc < kNumClasses; ++cc) {
        const uint32_t m = __ballot_sync(0xffffffffu, c == cc);
        if (c == cc) rank = __popc(m & lanemask_lt());
        if (lane == 0) s_wc[warp][cc] = __popc(m);
      }
      __syncthreads();
      if (c >= 0) {
        uint32_t before = s_run[c];
        for (uint32_t w = 0; w < warp; ++w) before += s_wc[w][c];
        const uint32_t id = pl.world <= 1 ? before + rank
                                          : plan_new_id(pl, c, before + rank - s_cstart[c]);
        perm[v] = id;
        inv[id] = v;
      }
      __syncthreads();
      if (threadIdx.x < kNumClasses) {
        uint32_t s = 0;
        for (int w = 0; w < W; ++w) s += s_wc[w][threadIdx.x];
        s_run[threadIdx.x] += s;
      }
      __syncthreads();
    }
  }
}

}  // namespace egs

namespace egs {

// ------------------------------------------ CSC transpose: radix sort ----
// The predecessor transpose (arena.cpp:56-74; the paper's CUSPARSE csr2csc,
// PAPER.md:529-530) is a STABLE sort of the (dst, src) pairs of the
// relabelled CSR by dst: within a column the sources keep CSR order, i.e.
// ascending, exactly the reference's stable transpose.  LSD radix sort with
// 8-bit digits; each pass is a stable counting sort:
//   k_radix_hist     per-tile digit histogram (tiles of kRadixTile pairs), written
//                    digit-major: hist[d * ntiles + tile]
//   dev_excl_scan    of the histogram = each (digit, tile)'s output offset
//   k_radix_scatter  warp w of a tile takes its kRadixSteps * 32 consecutive
//                    pairs in steps of 32; __match_any_sync groups a
//                    step's lanes by digit, per-warp digit counters give each
//                    pair its rank in (warp, step, lane) order = tile order,
//                    a prefix over warps per digit completes the tile rank.
constexpr int kRadixBits = 8;
constexpr int kRadixDigits = 1 << kRadixBits;
#ifndef EGS_RADIX_STEPS
#define EGS_RADIX_STEPS 8
#endif
constexpr int kRadixSteps = EGS_RADIX_STEPS;           // steps of 32 pairs per warp
constexpr uint32_t kRadixTile = kScanThreads * kRadixSteps;  // pairs per tile

__global__ void __launch_bounds__(kScanThreads)
    k_radix_hist(const uint32_t* key, uint64_t m, int shift, uint32_t* hist, uint32_t ntiles) {
  __shared__ unsigned int s_h[kRadixDigits];
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int d = threadIdx.x; d < kRadixDigits; d += kScanThreads) s_h[d] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)t * kRadixTile;
#pragma unroll 4
    for (int k = 0; k < kRadixSteps; ++k) {
      const uint64_t i = base + (uint64_t)k * kScanThreads + threadIdx.x;
      if (i < m) atomicAdd(&s_h[(key[i] >> shift) & (kRadixDigits - 1)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadixDigits; d += kScanThreads)
      hist[(uint64_t)d * ntiles + t] = s_h[d];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kScanThreads)
    k_radix_scatter(const uint32_t* key, const uint32_t* val, uint64_t m, int shift,
                    const uint32_t* off, uint32_t ntiles, uint32_t* key_out, uint32_t* val_out) {
  constexpr int W = kScanThreads / 32;
  __shared__ uint32_t s_wc[W][kRadixDigits];  // per-warp digit counts, then warp prefixes
  __shared__ uint32_t s_off[kRadixDigits];    // the tile's output offset per digit
  __shared__ uint32_t s_start[kRadixDigits];  // the digit's first position in the tile
  __shared__ uint32_t s_scan[33];
  __shared__ uint32_t s_key[kRadixTile], s_val[kRadixTile];  // the tile, locally sorted
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int i = threadIdx.x; i < W * kRadixDigits; i += kScanThreads) (&s_wc[0][0])[i] = 0;
    for (int d = threadIdx.x; d < kRadixDigits; d += kScanThreads)
      s_off[d] = off[(uint64_t)d * ntiles + t];
    __syncthreads();
    const uint64_t tbase = (uint64_t)t * kRadixTile;
    const uint64_t wbase = tbase + (uint64_t)warp * 32 * kRadixSteps;
    const uint32_t nt = (uint32_t)(m - tbase < kRadixTile ? m - tbase : kRadixTile);
    uint32_t k_[kRadixSteps], v_[kRadixSteps], r_[kRadixSteps];
    // every load of the warp's 512 pairs first: the ranking steps below
    // synchronise the warp, which the compiler does not move loads across
#pragma unroll
    for (int s = 0; s < kRadixSteps; ++s) {
      const uint64_t i = wbase + (uint64_t)s * 32 + lane;
      k_[s] = i < m ? __ldcs(key + i) : 0u;
      v_[s] = i < m ? __ldcs(val + i) : 0u;
    }
#pragma unroll
    for (int s = 0; s < kRadixSteps; ++s) {
      const uint64_t i = wbase + (uint64_t)s * 32 + lane;
      const bool in = i < m;
      const uint32_t d = in ? (k_[s] >> shift) & (kRadixDigits - 1) : 0u;
      // the lanes with my digit: one ballot per digit bit, and the valid mask
      uint32_t peers = __ballot_sync(0xffffffffu, in);
      if (!in) peers = ~peers;
#pragma unroll
      for (int b = 0; b < kRadixBits; ++b) {
        const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        peers &= ((d >> b) & 1u) ? bb : ~bb;
      }
      const uint32_t base = in ? s_wc[warp][d] : 0u;
      __syncwarp();
      if (in && (peers & lanemask_lt()) == 0) s_wc[warp][d] = base + __popc(peers);
      __syncwarp();
      r_[s] = base + __popc(peers & lanemask_lt());
    }
    __syncthreads();
    // per digit: warp prefixes and the tile total; then the digits' starts
    uint32_t tot = 0;
    for (int d = threadIdx.x; d < kRadixDigits; d += kScanThreads) {
      uint32_t acc = 0;
      for (int w = 0; w < W; ++w) {
        const uint32_t c = s_wc[w][d];
        s_wc[w][d] = acc;
        acc += c;
      }
      tot = acc;
    }
    static_assert(kRadixDigits == kScanThreads, "one digit per thread");
    const uint32_t start = block_excl_scan<uint32_t>(tot, s_scan, nullptr);
    s_start[threadIdx.x] = start;
    __syncthreads();
    // local sort into shared memory ...
#pragma unroll
    for (int s = 0; s < kRadixSteps; ++s) {
      const uint64_t i = wbase + (uint64_t)s * 32 + lane;
      if (i < m) {
        const uint32_t d = (k_[s] >> shift) & (kRadixDigits - 1);
        const uint32_t lp = s_start[d] + s_wc[warp][d] + r_[s];
        s_key[lp] = k_[s];
        s_val[lp] = v_[s];
      }
    }
    __syncthreads();
    // ... then out in local order: a digit's run goes to consecutive
    // addresses, so neighbouring threads write neighbouring words
    for (uint32_t lp = threadIdx.x; lp < nt; lp += kScanThreads) {
      const uint32_t kk = s_key[lp];
      const uint32_t d = (kk >> shift) & (kRadixDigits - 1);
      const uint32_t pos = s_off[d] + (lp - s_start[d]);
      key_out[pos] = kk;
      val_out[pos] = s_val[lp];
    }
    __syncthreads();
  }
}

}  // namespace egs
