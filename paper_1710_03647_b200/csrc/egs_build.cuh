// egs_build.cuh — device-side arena construction:
// the reference CSR (GameArena::build, proj/src/arena.cpp:17-78) is uploaded
// as-is and rebuilt on the device into the solver layout:
//
//   * vertices relabelled into six contiguous ranges by (owner, out-degree
//     class): the owner-sorted order of reorder_by_owner (arena.cpp:119-149;
//     PAPER.md:506-511) refined by row length, stable inside each range
//     (egs_scan.cuh k_class_tiles / k_class_place); with several ranks the
//     order is rank-major, each rank's block class-sorted (egs_part_plan);
//   * rows re-packed as edge records: 4-byte packed {dst | w << tbits} when
//     every weight fits beside the target bits, else 8-byte {u32 dst, i32 w}
//     (weights are validated to fit int32; arena.hpp:13 stores int64);
//   * the predecessor transpose (CSC, arena.cpp:56-74; the paper's CUSPARSE
//     csr2csc) built by a radix sort of (dst, src) pairs.
//
// Every kernel here runs once per arena upload, not per solve.
#pragma once

#include <climits>
#include <cstdint>

#include "egs_device.cuh"
#include "egs_types.cuh"

namespace egs {

// Row lengths in the new order (exclusive-scanned into offsets next); rows
// outside this rank's range [own_lo, own_hi) are empty here (multi-GPU: a
// rank stores its own rows only).
__global__ void k_row_lengths(uint32_t n, const uint32_t* inv, const uint64_t* off64,
                              uint32_t own_lo, uint32_t own_hi, uint32_t* deg_new) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += gridDim.x * blockDim.x) {
    const uint32_t o = inv[i];
    deg_new[i] = i >= own_lo && i < own_hi ? (uint32_t)(off64[o + 1] - off64[o]) : 0u;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) deg_new[n] = 0;
}

// Rows longer than kRelabelLong are not expanded by the warp that owns them
// with 31 other rows (a warp of 32 R-MAT rows of up to 2048 edges each held
// up a whole chunk: C3's relabel took 16 ms for 69 M edges, 20x C4's rate
// per edge).  The row-wise kernels queue them, k_long_prefix scans the
// queued rows' lengths, and the *_long kernels walk all their edges as one
// flat stream over the grid: a warp takes kRelabelLong consecutive edges --
// one binary search of the prefix, then at most one row boundary, as every
// queued row is longer than that.
constexpr uint32_t kRelabelLong = 256;

// pref[i] = edges of the queued rows before row i, pref[cnt] = all (one CTA)
__global__ void __launch_bounds__(1024)
    k_long_prefix(const uint32_t* list, const unsigned int* cnt_p, const uint64_t* off64,
                  uint64_t* pref) {
  __shared__ uint64_t s_warp[32];
  __shared__ uint64_t s_carry;
  const uint32_t cnt = *cnt_p, lane = lane_id(), warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < cnt; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    uint64_t x = 0;
    if (i < cnt) {
      const uint32_t o = list[i];
      x = off64[o + 1] - off64[o];
    }
    uint64_t inc = x;  // inclusive warp scan
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= (uint32_t)d) inc += y;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      uint64_t w = lane < (blockDim.x >> 5) ? s_warp[lane] : 0;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, w, d);
        if (lane >= (uint32_t)d) w += y;
      }
      s_warp[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const uint64_t before = s_carry + (warp ? s_warp[warp - 1] : 0) + inc - x;
    if (i < cnt) pref[i] = before;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry = before + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) pref[cnt] = s_carry;
}

// body(o, idx) for every edge idx of every queued row o, flat over the grid
template <class Body>
__device__ __forceinline__ void long_rows_flat(const uint32_t* list, const unsigned int* cnt_p,
                                               const uint64_t* off64, const uint64_t* pref,
                                               Body&& body) {
  const uint32_t cnt = *cnt_p;
  if (cnt == 0) return;
  const uint64_t total = pref[cnt];
  const uint32_t lane = lane_id();
  const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t g0 = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * kRelabelLong;
       g0 < total; g0 += nwarps * kRelabelLong) {
    uint32_t lo = 0, hi = cnt - 1;  // the row holding g0: last r with pref[r] <= g0
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (pref[mid] <= g0) lo = mid; else hi = mid - 1;
    }
    uint32_t r = lo;
    uint64_t r_end = pref[r + 1];
    uint32_t o = list[r];
    uint64_t b = off64[o];
    for (uint32_t s = 0; s < kRelabelLong / 32; ++s) {
      const uint64_t g = g0 + (uint64_t)s * 32 + lane;
      if (g >= total) break;
      if (g >= r_end) {  // (the next row: queued rows are longer than kRelabelLong)
        ++r;
        r_end = pref[r + 1];
        o = list[r];
        b = off64[o];
      }
      body(o, (uint32_t)(b + (g - pref[r])));
    }
  }
}

// Edge relabelling, pipelined with the chunked upload (egs_solver.cu
// build_arena): old rows [r0, r1) whose targets have arrived are copied to
// their relabelled slots, targets mapped through perm, with the (dst, src)
// pairs of the transpose; targets out of range set bit 2 of *bad.  A warp
// handles 32 rows and expands their edges as one flat coalesced stream
// (warp_expand), so short and long rows cost the same per edge.
__global__ void __launch_bounds__(256)
    k_relabel_targets(uint32_t n, uint32_t r0, uint32_t r1, const uint64_t* off64,
                      const uint32_t* dst, const uint32_t* perm, const uint32_t* off_new,
                      void* edge, uint32_t tbits, uint32_t* ckey, uint32_t* cval,
                      unsigned int* bad, uint32_t* longlist, unsigned int* longcnt,
                      uint32_t own_lo, uint32_t own_hi, bool key_at_orig) {
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int* ex = static_cast<int*>(edge);
  uint32_t* px = static_cast<uint32_t*>(edge);
  unsigned int flag = 0;
  for (uint32_t o0 = r0 + gw * 32; o0 < r1; o0 += nwarps * 32) {
    const uint32_t o = o0 + lane_id();
    uint32_t b = 0, e = 0, delta = 0, rn = 0;
    if (o < r1) {
      b = (uint32_t)off64[o];
      e = (uint32_t)off64[o + 1];
      rn = perm[o];
      delta = off_new[rn] - b;
      if (rn < own_lo || rn >= own_hi) {  // another rank's row (multi-GPU)
        e = b;
      } else if (e - b > kRelabelLong) {  // a hub: its edges go to the whole grid
        longlist[atomicAdd(longcnt, 1u)] = o;
        e = b;
      }
    }
    warp_expand(b, e, [&](bool valid, uint32_t idx, uint32_t owner_lane) {
      const uint32_t d = __shfl_sync(0xffffffffu, delta, owner_lane);
      const uint32_t src = __shfl_sync(0xffffffffu, rn, owner_lane);
      if (valid) {
        const uint32_t pos = idx + d;
        const uint32_t t0 = dst[idx];
        if (t0 >= n) flag |= 2u;
        const uint32_t t = perm[t0 < n ? t0 : 0];
        if (tbits)
          px[pos] = t;  // the weight half is or-ed in by k_relabel_weights
        else
          ex[2 * (size_t)pos] = (int)t;
        const uint32_t kp = key_at_orig ? idx : pos;  // (see k_csc_runs)
        ckey[kp] = t;
        cval[kp] = src;
      }
    });
  }
  flag = __reduce_or_sync(0xffffffffu, flag);
  if (lane_id() == 0 && flag) atomicOr(bad, flag);
}

// ... and the weight half once the weights of rows [r0, r1) have arrived
// (narrowed on the host to the narrowest of int8/int16/int32 that holds
// max |w|, range-checked there: arena.hpp:13 stores int64).
template <class W>
__global__ void __launch_bounds__(256)
    k_relabel_weights(uint32_t r0, uint32_t r1, const uint64_t* off64, const W* wn,
                      const uint32_t* perm, const uint32_t* off_new, void* edge,
                      uint32_t tbits, uint32_t* longlist, unsigned int* longcnt,
                      uint32_t own_lo, uint32_t own_hi) {
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int* ex = static_cast<int*>(edge);
  uint32_t* px = static_cast<uint32_t*>(edge);
  for (uint32_t o0 = r0 + gw * 32; o0 < r1; o0 += nwarps * 32) {
    const uint32_t o = o0 + lane_id();
    uint32_t b = 0, e = 0, delta = 0;
    if (o < r1) {
      b = (uint32_t)off64[o];
      e = (uint32_t)off64[o + 1];
      const uint32_t rn = perm[o];
      delta = off_new[rn] - b;
      if (rn < own_lo || rn >= own_hi) {
        e = b;
      } else if (e - b > kRelabelLong) {
        longlist[atomicAdd(longcnt, 1u)] = o;
        e = b;
      }
    }
    warp_expand(b, e, [&](bool valid, uint32_t idx, uint32_t owner_lane) {
      const uint32_t d = __shfl_sync(0xffffffffu, delta, owner_lane);
      if (valid) {
        if (tbits)  // after k_relabel_targets of the same rows (stream order)
          px[idx + d] |= (uint32_t)(int)wn[idx] << tbits;
        else
          ex[2 * (size_t)(idx + d) + 1] = (int)wn[idx];
      }
    });
  }
}

__global__ void __launch_bounds__(256)
    k_relabel_targets_long(uint32_t n, const uint32_t* longlist, const unsigned int* longcnt,
                           const uint64_t* pref, const uint64_t* off64, const uint32_t* dst,
                           const uint32_t* perm, const uint32_t* off_new, void* edge,
                           uint32_t tbits, uint32_t* ckey, uint32_t* cval, unsigned int* bad,
                           bool key_at_orig) {
  int* ex = static_cast<int*>(edge);
  uint32_t* px = static_cast<uint32_t*>(edge);
  unsigned int flag = 0;
  long_rows_flat(longlist, longcnt, off64, pref, [&](uint32_t o, uint32_t idx) {
    const uint32_t rn = perm[o];
    const uint32_t pos = idx + (off_new[rn] - (uint32_t)off64[o]);
    const uint32_t t0 = dst[idx];
    if (t0 >= n) flag |= 2u;
    const uint32_t t = perm[t0 < n ? t0 : 0];
    if (tbits)
      px[pos] = t;
    else
      ex[2 * (size_t)pos] = (int)t;
    const uint32_t kp = key_at_orig ? idx : pos;
    ckey[kp] = t;
    cval[kp] = rn;
  });
  if (flag) atomicOr(bad, flag);
}

template <class W>
__global__ void __launch_bounds__(256)
    k_relabel_weights_long(const uint32_t* longlist, const unsigned int* longcnt,
                           const uint64_t* pref, const uint64_t* off64, const W* wn,
                           const uint32_t* perm, const uint32_t* off_new, void* edge,
                           uint32_t tbits) {
  int* ex = static_cast<int*>(edge);
  uint32_t* px = static_cast<uint32_t*>(edge);
  long_rows_flat(longlist, longcnt, off64, pref, [&](uint32_t o, uint32_t idx) {
    const uint32_t d = off_new[perm[o]] - (uint32_t)off64[o];
    if (tbits)
      px[idx + d] |= (uint32_t)(int)wn[idx] << tbits;
    else
      ex[2 * (size_t)(idx + d) + 1] = (int)wn[idx];
  });
}

// Player-1 light rows (<= 32 edges) sorted by weight, ascending (ties by
// target), once per upload.  A player-1 row's order is free: its lift is a
// max (measure_ops.hpp:44-48) and no player-1 strategy is printed
// (extract_strategy, measure_ops.cpp:56-80, covers player 0 only; player-0
// rows keep the reference order).  Sorted, the first record holds the
// row's least weight, which is round 1's value (delta(0)(v) = max(0, -w_min)),
// and the certificate meets the likeliest good edges first (egs_solve.cuh).
// One warp per row: a 32-lane bitonic sort of the records as signed keys
// (packed: w in the high bits, so int32 order is (w, dst) order; wide:
// (w, dst) as an int64).  key[o] is the class of original row o
// (egs_scan.cuh k_class_tiles); class 3 = player-1 light.
// ascending bitonic sort of one value per lane over groups of G lanes
template <class K, uint32_t G = 32>
__device__ __forceinline__ K bitonic32(K x) {
  const uint32_t lane = lane_id() & (G - 1);
#pragma unroll
  for (uint32_t k = 2; k <= G; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      const K y = __shfl_xor_sync(0xffffffffu, x, j);
      const bool up = (lane & k) == 0, lower = (lane & j) == 0;
      x = (lower == up) ? (y < x ? y : x) : (y > x ? y : x);
    }
  }
  return x;
}

// sort the row (b, len) with groups of G lanes (lane index within the group);
// the group's first lane also mirrors the sorted first record into rec0[v]
template <uint32_t G>
__device__ __forceinline__ void sort_row(void* edge, uint32_t tbits, uint32_t b, uint32_t len,
                                         bool on, void* rec0, uint32_t v) {
  const uint32_t l = lane_id() & (G - 1);
  if (tbits) {
    int* rec = static_cast<int*>(edge) + b;
    const int x = bitonic32<int, G>(on && l < len ? rec[l] : INT32_MAX);
    if (on && l < len) rec[l] = x;
    if (on && l == 0) static_cast<int*>(rec0)[v] = x;
  } else {
    int2* rec = static_cast<int2*>(edge) + b;
    long long x = LLONG_MAX;
    if (on && l < len) {
      const int2 r = rec[l];
      x = ((long long)r.y << 32) | (long long)(uint32_t)r.x;
    }
    x = bitonic32<long long, G>(x);
    const int2 r = make_int2((int)(uint32_t)x, (int)(x >> 32));
    if (on && l < len) rec[l] = r;
    if (on && l == 0) static_cast<int2*>(rec0)[v] = r;
  }
}

// A warp takes two rows: one per half-warp when both have <= 16 edges (the
// common case), else one after the other with the whole warp.  Each row's
// first record after the sort -- its least weight, all that round 1 needs of
// a player-1 row (egs_solve.cuh round1_p1_light) -- is mirrored into rec0[v]
// (4 or 8 bytes per vertex, read coalesced, instead of a 32-byte sector of
// the row).
__global__ void __launch_bounds__(256)
    k_sort_p1_rows(uint32_t r0, uint32_t r1, const uint8_t* key, const uint32_t* perm,
                   const uint32_t* off_new, void* edge, uint32_t tbits, uint32_t own_lo,
                   uint32_t own_hi, void* rec0) {
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  const uint32_t lane = lane_id();
  for (uint32_t o0 = r0 + 2 * ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); o0 < r1;
       o0 += 2 * nwarps) {
    const uint32_t o = o0 + (lane >> 4);
    bool on = false;
    uint32_t b = 0, len = 0, v = 0;
    if (o < r1 && key[o] == (uint8_t)kP1L) {
      v = perm[o];
      if (v >= own_lo && v < own_hi) {
        b = off_new[v];
        len = off_new[v + 1] - b;
        on = len >= 2;
        if (len == 1 && (lane & 15u) == 0) {  // nothing to sort: mirror the record
          if (tbits)
            static_cast<int*>(rec0)[v] = static_cast<const int*>(edge)[b];
          else
            static_cast<int2*>(rec0)[v] = static_cast<const int2*>(edge)[b];
        }
      }
    }
    if (!__any_sync(0xffffffffu, on)) continue;
    if (!__any_sync(0xffffffffu, on && len > 16)) {
      sort_row<16>(edge, tbits, b, len, on, rec0, v);
    } else {
      for (uint32_t h = 0; h < 2; ++h) {  // warp-uniform
        const uint32_t bh = __shfl_sync(0xffffffffu, b, 16 * h);
        const uint32_t lh = __shfl_sync(0xffffffffu, len, 16 * h);
        const bool oh = __shfl_sync(0xffffffffu, on, 16 * h);
        const uint32_t vh = __shfl_sync(0xffffffffu, v, 16 * h);
        if (oh) sort_row<32>(edge, tbits, bh, lh, true, rec0, vh);
      }
    }
  }
}

// Transpose built chunk by chunk while the upload runs (single-rank build,
// egs_solver.cu build_arena).  Each target chunk's (target, source) pairs sit
// at their original edge positions; once sorted by target (stably: original
// order within a target), every element gets its slot inside its column
// relative to the column start -- the column's edges from earlier chunks
// (cnt) plus its rank in this chunk's run of that target.  After the last
// chunk the column offsets are the scan of cnt and one scatter places every
// source.  A column lists its sources in original edge order, which for a
// CSR is ascending original source id.
// Heads of the runs of the sorted chunk: rb[t] = {run start, edges of t in
// earlier chunks}.
__global__ void k_csc_runs(const uint32_t* key, uint64_t len, const uint32_t* cnt, uint2* rb) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += stride) {
    const uint32_t t = key[i];
    if (i == 0 || key[i - 1] != t) rb[t] = make_uint2((uint32_t)i, cnt[t]);
  }
}
// rel[i] = the element's slot in its column; the run's last element adds the
// run to cnt (read above only by the heads, so no element races its update)
__global__ void k_csc_rel(const uint32_t* key, uint64_t len, const uint2* rb, uint32_t* cnt,
                          uint32_t* rel) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += stride) {
    const uint32_t t = key[i];
    const uint2 h = rb[t];
    const uint32_t r = h.y + (uint32_t)(i - h.x);
    rel[i] = r;
    if (i + 1 == len || key[i + 1] != t) cnt[t] = r + 1;
  }
}
// csrc[coff[t] + rel] = source.  A plain scatter writes 4 bytes per 32-byte
// sector (a chunk holds ~one edge per column): 5.6 ms at C4.  Instead each
// CTA assembles kMergeSpan consecutive output slots in shared memory and
// stores them coalesced.  Within one chunk's sorted pairs the slot
// pos(i) = coff[key[i]] + rel[i] strictly increases with i (rel counts up
// inside a run, and a column's slots end before the next column's start), so
// the pairs landing in [p0, p1) are one contiguous range per chunk: two
// binary searches, one lane per chunk.  Each pair is read once, hubs
// included.
constexpr uint32_t kMergeSpan = 8192;
constexpr int kMaxChunks = 32;
struct ChunkStarts {
  uint64_t e[kMaxChunks + 1];  // chunk k's sorted pairs: [e[k], e[k+1])
  int nch;
};
// first i in [lo, hi) with coff[key[i]] + rel[i] >= p
__device__ __forceinline__ uint64_t lower_slot(const uint32_t* key, const uint32_t* rel,
                                               const uint32_t* coff, uint64_t lo, uint64_t hi,
                                               uint64_t p) {
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if ((uint64_t)coff[key[mid]] + rel[mid] < p)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}
__global__ void __launch_bounds__(512)
    k_csc_merge(const uint32_t* key, const uint32_t* val, const uint32_t* rel, uint64_t m,
                const uint32_t* coff, ChunkStarts cs, uint32_t* csrc) {
  __shared__ uint32_t slot[kMergeSpan];
  __shared__ uint64_t rlo[kMaxChunks], rhi[kMaxChunks];
  for (uint64_t p0 = (uint64_t)blockIdx.x * kMergeSpan; p0 < m;
       p0 += (uint64_t)gridDim.x * kMergeSpan) {
    const uint64_t p1 = min(m, p0 + (uint64_t)kMergeSpan);
    if (threadIdx.x < 2u * cs.nch) {
      const int k = threadIdx.x >> 1;
      if (threadIdx.x & 1)
        rhi[k] = lower_slot(key, rel, coff, cs.e[k], cs.e[k + 1], p1);
      else
        rlo[k] = lower_slot(key, rel, coff, cs.e[k], cs.e[k + 1], p0);
    }
    __syncthreads();
    for (int k = 0; k < cs.nch; ++k)
      for (uint64_t i = rlo[k] + threadIdx.x; i < rhi[k]; i += blockDim.x)
        slot[coff[key[i]] + rel[i] - p0] = val[i];
    __syncthreads();
    for (uint64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) csrc[p] = slot[p - p0];
    __syncthreads();
  }
}

// CSC column offsets from the dst-sorted keys: coff[t] = first j with
// key[j] >= t, coff[n] = m.
__global__ void k_col_offsets(uint32_t n, uint64_t m, const uint32_t* key,
                              uint32_t* coff) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= m; j += stride) {
    const uint32_t k = j < m ? key[j] : n;
    const int64_t prev = j > 0 ? (int64_t)key[j - 1] : -1;
    for (int64_t t = prev + 1; t <= (int64_t)k; ++t) coff[t] = (uint32_t)j;
  }
}

// ---------------------------------------------------- measure I/O ----
// out[old] = widen(f[perm[old]]): device values (u32/u64, top = all ones)
// back to the reference raw encoding (INT64_MAX = top, energy.hpp:16).
template <class V>
__global__ void k_export(uint32_t n, const V* f, const uint32_t* perm, int64_t* out) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += gridDim.x * blockDim.x) {
    const V x = f[perm[v]];
    out[v] = x == Top<V>::v ? INT64_MAX : static_cast<int64_t>(x);
  }
}

// 32-bit values in original ids, top kept as all ones (widened on the host:
// egs_internal_widen_u32)
__global__ void k_export_u32(uint32_t n, const uint32_t* f, const uint32_t* perm, uint32_t* out) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += gridDim.x * blockDim.x)
    out[v] = f[perm[v]];
}

// out[v] = widen(f[v]) in relabelled ids (the debug_checks fixpoint test of
// a solve's own result).
template <class V>
__global__ void k_widen(uint32_t n, const V* f, int64_t* out) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += gridDim.x * blockDim.x) {
    const V x = f[v];
    out[v] = x == Top<V>::v ? INT64_MAX : static_cast<int64_t>(x);
  }
}

// fnew[perm[old]] = fin[old] (int64, raw encoding) for the verifier.
__global__ void k_import(uint32_t n, const int64_t* fin, const uint32_t* perm,
                         int64_t* fnew) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += gridDim.x * blockDim.x)
    fnew[perm[v]] = fin[v];
}

// epm_condition_holds for every vertex (measure_ops.cpp:17-31) on a raw int64
// measure in relabelled ids, with the reference's uncapped ⊖ (energy.hpp:
// 20-31): player 0 needs some edge with f(v) >= f(t) ⊖ w, player 1 needs it
// on every edge.  One warp per vertex so hub rows are read cooperatively.
// *bad counts violating vertices; *overflow flags a raw_ominus overflow.
__device__ __forceinline__ int64_t ominus_raw(int64_t ft, int32_t w, int* overflow) {
  if (ft == INT64_MAX) return INT64_MAX;
  if (w < 0 && ft > INT64_MAX + (int64_t)w) {
    atomicExch(overflow, 1);
    return INT64_MAX;
  }
  const int64_t c = ft - w;
  return c < 0 ? 0 : c;
}

__global__ void __launch_bounds__(256)
    k_epm(Graph g, const int64_t* f, unsigned long long* bad, int* overflow) {
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  unsigned long long nb = 0;
  for (uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < g.n; v += nwarps) {
    const int64_t fv = f[v];
    const bool p0 = v < g.rb[kP1L];
    const uint32_t b = g.off[v], e = g.off[v + 1];
    bool ok = !p0;
    for (uint32_t i0 = b; i0 < e; i0 += 32) {
      const uint32_t i = i0 + lane_id();
      bool sat = true;  // f(v) >= f(t) ⊖ w on this edge
      if (i < e) {
        const int2 r = edge_at(g, i);
        sat = fv >= ominus_raw(f[r.x], r.y, overflow);
      }
      if (p0) {
        if (__any_sync(0xffffffffu, i < e && sat)) {
          ok = true;
          break;
        }
      } else if (!__all_sync(0xffffffffu, sat)) {
        ok = false;
        break;
      }
    }
    if (!ok && lane_id() == 0) ++nb;
  }
  if (nb) atomicAdd(bad, nb);
}

// Fixpoint check of a raw int64 measure (relabelled ids): delta(f)(v) ==
// f(v) for every vertex, with the lift's cap (`> credit_cap -> top`,
// measure_ops.hpp:51).  The least progress measure is the least fixpoint of
// this lift, so a solve result must pass it exactly; *bad counts vertices
// where the lift differs from f.  One warp per vertex.
__global__ void __launch_bounds__(256)
    k_fixpoint(Graph g, const int64_t* f, unsigned long long* bad) {
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  unsigned long long nb = 0;
  for (uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < g.n; v += nwarps) {
    const bool p0 = v < g.rb[kP1L];
    const uint32_t b = g.off[v], e = g.off[v + 1];
    int64_t acc = p0 ? INT64_MAX : 0;
    for (uint32_t i = b + lane_id(); i < e; i += 32) {
      const int2 r = edge_at(g, i);
      const int64_t ft = f[r.x];
      int64_t c = ft == INT64_MAX ? INT64_MAX : ft - (int64_t)r.y;
      if (c != INT64_MAX) {
        c = c < 0 ? 0 : c;
        c = c > g.cap ? INT64_MAX : c;
      }
      acc = p0 ? (c < acc ? c : acc) : (c > acc ? c : acc);
    }
#pragma unroll
    for (int sft = 16; sft > 0; sft >>= 1) {
      const int64_t y = __shfl_xor_sync(0xffffffffu, acc, sft);
      acc = p0 ? (y < acc ? y : acc) : (y > acc ? y : acc);
    }
    if (lane_id() == 0 && acc != f[v]) ++nb;
  }
  if (nb) atomicAdd(bad, nb);
}

// The transpose holds exactly the CSR's edges: an order-free fingerprint,
// sum[0] over the CSR rows and sum[1] over the CSC columns of
// mix(source, target), plus sum[2] = columns whose offsets decrease.  One warp
// per vertex (debug checks only).
__device__ __forceinline__ unsigned long long edge_mix(uint32_t s, uint32_t t) {
  unsigned long long x = ((unsigned long long)s << 32 | t) + 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__global__ void __launch_bounds__(256)
    k_csc_check(Graph g, unsigned long long* sum) {
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  unsigned long long a = 0, b = 0, bad = 0;
  for (uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < g.n; v += nwarps) {
    for (uint32_t i = g.off[v] + lane_id(); i < g.off[v + 1]; i += 32)
      a += edge_mix(v, (uint32_t)edge_at(g, i).x);
    const uint32_t cb = g.coff[v], ce = g.coff[v + 1];
    if (lane_id() == 0 && ce < cb) ++bad;
    for (uint32_t j = cb + lane_id(); j < ce; j += 32) b += edge_mix(g.csrc[j], v);
  }
  if (a) atomicAdd(sum, a);
  if (b) atomicAdd(sum + 1, b);
  if (bad) atomicAdd(sum + 2, bad);
}

// sum over v of edge_mix(v, f[v]) (wrapping): egs_part_digest
template <class V>
__global__ void k_digest(uint32_t n, const V* f, unsigned long long* out) {
  unsigned long long h = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint64_t x = (uint64_t)f[v];
    h += edge_mix(v, (uint32_t)x) ^ edge_mix((uint32_t)(x >> 32), ~v);
  }
#pragma unroll
  for (int sft = 16; sft > 0; sft >>= 1) h += __shfl_xor_sync(0xffffffffu, h, sft);
  if (lane_id() == 0 && h) atomicAdd(out, h);
}

// ---------------------------------------------- solution output ----
// write_solution(make_solution(...)) (io.cpp:178-210) on the device.  The
// strategy of a finite player-0 vertex is the FIRST successor in row order
// with f(v) >= f(t) ⊖ w (extract_strategy, measure_ops.cpp:56-80); rows keep
// their input order through the relabelling, so the first witness of the
// relabelled row is the reference's.  strat[old id] = old target or ~0u.
constexpr uint32_t kNoTarget = 0xFFFFFFFFu;

template <class V>
__device__ __forceinline__ int64_t raw_of(V x) {
  return x == Top<V>::v ? INT64_MAX : static_cast<int64_t>(x);
}

template <class V>
__global__ void __launch_bounds__(256)
    k_strategy(Graph g, const V* f, const uint32_t* inv, uint32_t* strat, int* err) {
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < g.n; v += nwarps) {
    const int64_t fv = raw_of<V>(f[v]);
    uint32_t target = kNoTarget;
    if (v < g.rb[kP1L] && fv != INT64_MAX) {
      const uint32_t b = g.off[v], e = g.off[v + 1];
      for (uint32_t i0 = b; i0 < e; i0 += 32) {
        const uint32_t i = i0 + lane_id();
        bool sat = false;
        int2 r = make_int2(0, 0);
        if (i < e) {
          r = edge_at(g, i);
          sat = fv >= ominus_raw(raw_of<V>(f[r.x]), r.y, err);
        }
        const uint32_t m = __ballot_sync(0xffffffffu, sat);
        if (m) {
          const int src = __ffs(m) - 1;
          target = inv[__shfl_sync(0xffffffffu, r.x, src)];
          break;
        }
      }
      if (target == kNoTarget && lane_id() == 0) atomicExch(err, 2);  // NoWitnessError
    }
    if (lane_id() == 0) strat[inv[v]] = target;
  }
}

__device__ __forceinline__ uint32_t dec_digits(uint64_t x) {
  uint32_t d = 1;
  while (x >= 10) {
    x /= 10;
    ++d;
  }
  return d;
}
__device__ __forceinline__ void dec_write(char* out, uint64_t x, uint32_t d) {
  for (uint32_t k = d; k > 0; --k) {
    out[k - 1] = (char)('0' + x % 10);
    x /= 10;
  }
}

// Line lengths "<id> <value|T>[ <target>]\n" by original id.
template <class V>
__global__ void k_line_len(uint32_t n, const V* f, const uint32_t* perm, const uint32_t* strat,
                           unsigned long long* len) {
  for (uint32_t o = blockIdx.x * blockDim.x + threadIdx.x; o < n; o += gridDim.x * blockDim.x) {
    const V x = f[perm[o]];
    uint64_t l = dec_digits(o) + 2 + (x == Top<V>::v ? 1 : dec_digits(x));
    if (strat[o] != kNoTarget) l += 1 + dec_digits(strat[o]);
    len[o] = l;
  }
}

template <class V>
__global__ void k_format(uint32_t n, const V* f, const uint32_t* perm, const uint32_t* strat,
                         const unsigned long long* pos, char* text) {
  for (uint32_t o = blockIdx.x * blockDim.x + threadIdx.x; o < n; o += gridDim.x * blockDim.x) {
    char* p = text + pos[o];
    uint32_t d = dec_digits(o);
    dec_write(p, o, d);
    p += d;
    *p++ = ' ';
    const V x = f[perm[o]];
    if (x == Top<V>::v) {
      *p++ = 'T';
    } else {
      d = dec_digits(x);
      dec_write(p, x, d);
      p += d;
    }
    if (strat[o] != kNoTarget) {
      *p++ = ' ';
      d = dec_digits(strat[o]);
      dec_write(p, strat[o], d);
      p += d;
    }
    *p = '\n';
  }
}

}  // namespace egs
