// egs_solve.cuh — the persistent value-iteration kernel (one launch per
// solve, device-side convergence; no host round trip between rounds).
//
// It restates the reference solve path (/root/reference/proj):
//   seed phase        solver_par.cpp:368-387 / solver_seq.cpp:136-154
//   lift phases       raw_lift (measure_ops.hpp:32-52) applied as the rounds
//                     of solve_frontier (solver_par.cpp:389-417, sparse) or
//                     solve_sweep (solver_par.cpp:205-228, dense), with the
//                     clamped store `cand > old` (solver_par.cpp:216,399)
//   activation phase  predecessor activation + dedup (solver_par.cpp:402-410)
//                     and the top filter of the gather (solver_par.cpp:305-311)
//   certificate       DESIGN.md §3: proves a set of vertices losing for
//                     player 0 so their value jumps to top instead of
//                     climbing to credit_cap one weight at a time.
//   termination       a lift round that raises nothing (solver_par.cpp:170-194)
//
// Vertices are relabelled on the device (egs_build.cuh) into six contiguous
// ranges: player 0 light / medium / heavy, then player 1 light / medium /
// heavy (the owner-sorted order of reorder_by_owner, arena.cpp:119-149,
// PAPER.md:506-511, refined by out-degree).  Light rows (<= 32 edges) are
// lifted by one thread, medium rows (<= 4096) by one warp, heavy rows (the
// R-MAT hubs) by one CTA, so warps never mix min and max and never wait on
// one long row.
//
// Phases are separated by grid-wide barriers (cooperative launch).  Rounds
// are synchronous (Jacobi): lifts read the measure of the previous round
// and stage raised values, which a commit phase publishes; a round that
// raises nothing has reached the least fixpoint, exactly as the reference's
// `changed` latch decides (solver_par.cpp:170-194).  Jacobi iterates keep
// the per-round climb of losing vertices regular, which is what lets the
// certificate prove the whole losing region in one attempt.
#pragma once

#include <cooperative_groups.h>

#include <cstdint>
#include <type_traits>

#include "egs_device.cuh"
#include "egs_types.cuh"

#ifndef EGS_EDGE_BYTES
#define EGS_EDGE_BYTES 8
#endif
#ifndef EGS_FMT_NS
#define EGS_FMT_NS e8
#endif

namespace egs {
namespace EGS_FMT_NS {

namespace cg = cooperative_groups;

// ---- the edge-record format of this translation unit (egs_types.cuh)
#if EGS_EDGE_BYTES == 4
using ERec = uint32_t;
__device__ __forceinline__ int2 dec(const Graph& g, ERec r) { return edge_dec(r, g.tbits); }
__device__ __forceinline__ ERec enc(const Graph& g, int2 e) {
  return (uint32_t)e.x | ((uint32_t)e.y << g.tbits);
}
__device__ __forceinline__ int rec_w(const Graph& g, ERec r) { return (int)r >> g.tbits; }
#else
using ERec = int2;
__device__ __forceinline__ int2 dec(const Graph&, ERec r) { return r; }
__device__ __forceinline__ ERec enc(const Graph&, int2 e) { return e; }
__device__ __forceinline__ int rec_w(const Graph&, ERec r) { return r.y; }
#endif
__device__ __forceinline__ const ERec* erecs(const Graph& g) {
  return static_cast<const ERec*>(g.edge);
}
// streaming (evict-first) load of edge i, decoded
__device__ __forceinline__ int2 ld_rec(const Graph& g, uint32_t i) {
  return dec(g, __ldcs(erecs(g) + i));
}
template <class V>
__device__ __forceinline__ ERec* wit_of(const SolveParams<V>& p) {
  return static_cast<ERec*>(p.wit);
}
template <class V>
__device__ __forceinline__ int2 ld_wit(const SolveParams<V>& p, uint32_t v) {
  return dec(p.g, ldcg(wit_of(p) + v));
}
template <class V>
__device__ __forceinline__ void st_wit(const SolveParams<V>& p, uint32_t v, int2 e) {
  stcg(wit_of(p) + v, enc(p.g, e));
}

// ---- class ranges and the owned vertex range (multi-GPU)
__device__ __forceinline__ int size_class(const Graph& g, uint32_t v) {
  if (v < g.rb[kP1L]) return v >= g.rb[kP0H] ? 2 : v >= g.rb[kP0M] ? 1 : 0;
  return v >= g.rb[kP1H] ? 2 : v >= g.rb[kP1M] ? 1 : 0;
}
// i-th vertex of the union of the player-0 and player-1 ranges of class c
__device__ __forceinline__ uint32_t class_item(const Graph& g, int c, uint32_t i) {
  const uint32_t n0 = g.rb[c + 1] - g.rb[c];
  return i < n0 ? g.rb[c] + i : g.rb[c + 3] + (i - n0);
}
__device__ __forceinline__ uint32_t class_size(const Graph& g, int c) {
  return (g.rb[c + 1] - g.rb[c]) + (g.rb[c + 4] - g.rb[c + 3]);
}
template <class V>
__device__ __forceinline__ bool owned(const SolveParams<V>& p, uint32_t v) {
  return v >= p.own_lo && v < p.own_hi;
}
template <class V>
__device__ __forceinline__ uint32_t clip_lo(const SolveParams<V>& p, uint32_t lo) {
  return lo > p.own_lo ? lo : p.own_lo;
}
template <class V>
__device__ __forceinline__ uint32_t clip_hi(const SolveParams<V>& p, uint32_t hi) {
  return hi < p.own_hi ? hi : p.own_hi;
}

// ---- replicated writes (multi-GPU): a value or bit a rank produces for its
// own vertices goes to its own replica and to every peer's (NVLink peer
// stores / system-scope atomics); with one rank these are plain writes.
template <class V, class T>
__device__ __forceinline__ T* peer_of(const SolveParams<V>& p, int q, T* local) {
  return reinterpret_cast<T*>(p.xpeer[q] + (reinterpret_cast<char*>(local) - p.xbase));
}
template <class V>
__device__ __forceinline__ void bits_or(const SolveParams<V>& p, uint32_t* word, uint32_t m) {
  if (p.world == 1) {
    atomicOr(word, m);
    return;
  }
  for (int q = 0; q < p.world; ++q) atomicOr_system(peer_of(p, q, word), m);
}
template <class V>
__device__ __forceinline__ void set_bit(const SolveParams<V>& p, uint32_t* bm, uint32_t v) {
  bits_or(p, bm + (v >> 5), 1u << (v & 31u));
}
// the bits of bitmap word w that are this rank's vertices (the replicated
// bitmaps carry every rank's)
template <class V>
__device__ __forceinline__ uint32_t own_mask(const SolveParams<V>& p, uint32_t w) {
  if (p.world == 1) return ~0u;
  const uint32_t lo = w << 5;
  if (lo >= p.own_lo && lo + 32 <= p.own_hi) return ~0u;
  uint32_t m = 0;
  for (uint32_t i = 0; i < 32; ++i) m |= (uint32_t)(lo + i >= p.own_lo && lo + i < p.own_hi) << i;
  return m;
}
template <class V>
__device__ __forceinline__ void f_put(const SolveParams<V>& p, uint32_t v, V x) {
  stcg(p.f + v, x);
  if (p.world > 1)
    for (int q = 0; q < p.world; ++q)
      if (q != p.rank) stcg(peer_of(p, q, p.f + v), x);
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t vload(const volatile unsigned int* p) { return *p; }

// Per-CTA time spent in the sub-phases of a lift phase (thread 0 of each
// CTA adds its own wall time; divide by the grid size for a per-CTA mean).
// Only under EGS_TRACE (p.trace set): off the solve path otherwise.
struct SubTimer {
  unsigned long long* ctr;
  unsigned long long t;
  bool on;
  __device__ SubTimer(unsigned long long* c, bool enabled) : ctr(c), t(0), on(enabled) {
    if (on && threadIdx.x == 0) t = globaltimer();
  }
  __device__ void lap(int k) {
    if (on && threadIdx.x == 0) {
      const unsigned long long now = globaltimer();
      atomicAdd(ctr + k, now - t);
      t = now;
    }
  }
};

// Per-thread event counts of the current phase (u32: one phase touches every
// row / edge at most once, so a warp's sum stays below 2^32).
struct Local {
  unsigned int lifts = 0, apps = 0, edges = 0, witness = 0, act = 0, certified = 0,
               pops = 0, cert_scanned = 0, cert_edges = 0, visits = 0;
  unsigned int phase_count = 0;  // per-phase sum (changed / removed / seeds)
  unsigned int pushed = 0;       // frontier entries added by a sparse lift's pushes
};
constexpr int kLocalCounters = 10;

// Counters never cross a grid barrier on their own.  A warp reduces its
// lanes' counts (REDUX) and lane 0 adds them to per-CTA shared accumulators
// -- no __syncthreads, no global atomics inside a phase:
//   g_stats   the SolveReport statistics, added to p.ctr once per CTA at
//             kernel exit (stats_exit);
//   g_psum    the phase sums the control flow reads (changed / removed /
//             frontier sizes), one per Scratch::sum slot of the current
//             phase, added to it by end_phase_flush right before the grid
//             barrier (one global atomic per CTA and nonzero slot).
// g_slot_base is the current phase's Scratch::sum row; every warp writes it
// (the same value) before its first flush of the phase, so a read after a
// warp's own write is always the current phase's row.  (compute-sanitizer
// racecheck reports these same-value writes against other warps' reads as
// a shared-memory hazard: benign -- the row changes only across the grid
// barrier that ends a phase.  Deriving the slot from the address instead
// removed the report but cost C4 +28 us in the certificate's dense pass, a
// register-allocation change of the whole kernel.)
__shared__ unsigned long long g_stats[kLocalCounters];
__shared__ unsigned int g_psum[4];
__shared__ unsigned int* g_slot_base;

__device__ __forceinline__ void set_phase_slot(unsigned int* slot) {
  if (lane_id() == 0) g_slot_base = slot;
  __syncwarp();
}

__device__ __forceinline__ void stats_init() {
  if (threadIdx.x < (unsigned)kLocalCounters) g_stats[threadIdx.x] = 0ull;
  if (threadIdx.x < 4u) g_psum[threadIdx.x] = 0u;
  __syncthreads();
}

__device__ __forceinline__ void stats_exit(unsigned long long* ctr) {
  __syncthreads();
  if (threadIdx.x < (unsigned)kLocalCounters && g_stats[threadIdx.x])
    atomicAdd(ctr + threadIdx.x, g_stats[threadIdx.x]);
}

// Block-wide, before the grid barrier that ends a phase.
__device__ __forceinline__ void end_phase_flush() {
  __syncthreads();
  if (threadIdx.x < 4u) {
    const unsigned int v = g_psum[threadIdx.x];
    if (v) {
      atomicAdd(g_slot_base + threadIdx.x, v);
      g_psum[threadIdx.x] = 0u;
    }
  }
}

// Warp-wide flush of the phase's counters: phase_count goes to the phase sum
// slot `dst`, pushed to `dst2` (both in the current phase's Scratch::sum
// row).  Warp-uniform; every lane of the warp calls it.
__device__ __forceinline__ void block_flush(Local& L, unsigned int* dst,
                                            unsigned int* dst2 = nullptr) {
  constexpr int K = kLocalCounters + 2;  // + phase_count, pushed
  unsigned int v[K] = {L.lifts, L.apps,      L.edges,        L.witness,
                       L.act,   L.certified, L.pops,         L.cert_scanned,
                       L.cert_edges, L.visits, L.phase_count, L.pushed};
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = __reduce_add_sync(0xffffffffu, v[k]);
  if (lane_id() == 0) {
#pragma unroll
    for (int k = 0; k < kLocalCounters; ++k)
      if (v[k]) atomicAdd(&g_stats[k], (unsigned long long)v[k]);
    if (v[kLocalCounters]) atomicAdd(&g_psum[dst - g_slot_base], v[kLocalCounters]);
    if (v[kLocalCounters + 1] && dst2)
      atomicAdd(&g_psum[dst2 - g_slot_base], v[kLocalCounters + 1]);
  }
  L = Local();
}

// ============================================================== lifts ====
// The lift of one vertex: delta(f, v) = min (player 0) / max (player 1) over
// its row of f(t) ⊖ w, capped (raw_lift, measure_ops.hpp:32-52).  Returns
// whether the value rose.  Player 0 first tests its witness edge (the argmin
// of its last lift): values only rise, so while f(v) >= f(t) ⊖ w holds for
// it the lift cannot raise f(v) and the row is not read (the GPU analogue of
// the count(v) of Alg. 1, solver_seq.cpp:186-199).

// A raised value is staged for the round's commit (Jacobi rounds), or, in a
// sparse round, stored in place with atomicMax -- the in-place atomic store
// of solve_frontier (solver_par.cpp:399) -- and then true iff it rose.
template <class V, bool INPLACE>
__device__ __forceinline__ bool store_raise(const SolveParams<V>& p, uint32_t v, V acc, V old) {
  if (!(acc > old)) return false;
  if (!INPLACE) {
    stcg(p.stage + v, acc);
    return true;
  }
  bool up;
  if (sizeof(V) == 8)
    up = atomicMax(reinterpret_cast<unsigned long long*>(p.f + v), (unsigned long long)acc) <
         (unsigned long long)acc;
  else
    up = atomicMax(reinterpret_cast<unsigned int*>(p.f + v), (unsigned int)acc) < (unsigned int)acc;
  // only the owner writes v, once per sparse round: the peers' replicas take
  // the raised value with a plain store
  if (up && p.world > 1)
    for (int q = 0; q < p.world; ++q)
      if (q != p.rank) stcg(peer_of(p, q, p.f + v), acc);
  return up;
}

// ---- one thread per row (light rows)
#ifndef EGS_LIFT_CHUNK
#define EGS_LIFT_CHUNK 8
#endif
constexpr int kChunk = EGS_LIFT_CHUNK;  // edges whose gathers a thread keeps in flight

template <class V, bool P0, bool INPLACE = false>
__device__ __forceinline__ bool lift_thread(const SolveParams<V>& p, uint32_t v,
                                            Local& L) {
  constexpr V TOP = Top<V>::v;
  ++L.visits;
  const V old = ldcg(p.f + v);
  if (old == TOP) return false;
  if (P0) {
    const int2 we = ld_wit(p, v);
    if (old >= ominus_cap<V>(gather(p.f + we.x), we.y, p.g.cap)) {
      ++L.witness;
      return false;
    }
  }
  const uint32_t b = __ldg(p.g.off + v), e = __ldg(p.g.off + v + 1);
  ++L.apps;
  L.edges += e - b;
  V acc = P0 ? TOP : V(0);
  int2 best = make_int2(0, 0);
  // Branch-free chunks: indices past the row end re-read its last edge
  // (a duplicate cannot change a min or a max), so all loads of a chunk
  // issue back to back before the first use.
  for (uint32_t i = b; i < e; i += kChunk) {
    int2 r[kChunk];
#pragma unroll
    for (int k = 0; k < kChunk; ++k) r[k] = ld_rec(p.g, min(i + k, e - 1));
    V c[kChunk];
#pragma unroll
    for (int k = 0; k < kChunk; ++k) c[k] = gather(p.f + r[k].x);
#pragma unroll
    for (int k = 0; k < kChunk; ++k) {
      const V x = ominus_cap<V>(c[k], r[k].y, p.g.cap);
      if (P0) {
        // argmin; among equal values prefer a player-0 target (see round 1)
        const bool tp1 = (uint32_t)r[k].x >= p.g.rb[kP1L];
        if (x < acc || (k == 0 && i == b) ||
            (x == acc && !tp1 && (uint32_t)best.x >= p.g.rb[kP1L])) {
          acc = x;
          best = r[k];
        }
      } else {
        acc = x > acc ? x : acc;
      }
    }
    if (P0 ? acc == V(0) : acc == TOP) break;  // raw_lift early exits (:41,46)
  }
  if (P0) st_wit(p, v, best);
  if (store_raise<V, INPLACE>(p, v, acc, old)) {
    ++L.lifts;
    return true;
  }
  return false;
}

// ---- one warp per row (medium rows).  Warp-uniform.
template <class V, bool P0, bool INPLACE = false>
__device__ __forceinline__ bool lift_warp(const SolveParams<V>& p, uint32_t v,
                                          Local& L) {
  constexpr V TOP = Top<V>::v;
  const uint32_t lane = lane_id();
  if (lane == 0) ++L.visits;
  const V old = ldcg(p.f + v);
  if (old == TOP) return false;
  if (P0) {
    bool sat = false;
    if (lane == 0) {
      const int2 we = ld_wit(p, v);
      sat = old >= ominus_cap<V>(gather(p.f + we.x), we.y, p.g.cap);
    }
    if (__shfl_sync(0xffffffffu, sat, 0)) {
      if (lane == 0) ++L.witness;
      return false;
    }
  }
  const uint32_t b = __ldg(p.g.off + v), e = __ldg(p.g.off + v + 1);
  if (lane == 0) {
    ++L.apps;
    L.edges += e - b;
  }
  V acc = P0 ? TOP : V(0);
  int2 best = make_int2(0, 0);
  bool have = false;
  for (uint32_t i0 = b; i0 < e; i0 += 128) {
    int2 r[4];
    V c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t i = i0 + k * 32 + lane;
      if (i < e) r[k] = ld_rec(p.g, i);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t i = i0 + k * 32 + lane;
      if (i < e) c[k] = ominus_cap<V>(gather(p.f + r[k].x), r[k].y, p.g.cap);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t i = i0 + k * 32 + lane;
      if (i < e) {
        if (P0) {
          if (!have || c[k] < acc) {
            acc = c[k];
            best = r[k];
            have = true;
          }
        } else {
          acc = c[k] > acc ? c[k] : acc;
        }
      }
    }
    const V red = P0 ? warp_min(acc) : warp_max(acc);
    if (P0 ? red == V(0) : red == TOP) break;
  }
  const V res = P0 ? warp_min(acc) : warp_max(acc);
  bool raised = false;
  if (P0) {
    const uint32_t m = __ballot_sync(0xffffffffu, have && acc == res);
    const int src = __ffs(m) - 1;
    best.x = __shfl_sync(0xffffffffu, best.x, src);
    best.y = __shfl_sync(0xffffffffu, best.y, src);
  }
  if (lane == 0) {
    if (P0) st_wit(p, v, best);
    if (store_raise<V, INPLACE>(p, v, res, old)) {
      ++L.lifts;
      raised = true;
    }
  }
  return __shfl_sync(0xffffffffu, raised, 0);
}

// ---- one CTA per row (heavy rows).  Block-uniform.
template <class V>
struct BlockScratch {
  V val[kWarps];
  int2 rec[kWarps];
  unsigned int red[kWarps];
  unsigned int item;
  int flag;
};

template <class V, bool P0, bool INPLACE = false>
__device__ __forceinline__ bool lift_block(const SolveParams<V>& p, uint32_t v,
                                           Local& L, BlockScratch<V>& s) {
  constexpr V TOP = Top<V>::v;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) ++L.visits;
  const V old = ldcg(p.f + v);
  if (old == TOP) return false;
  if (P0) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const int2 we = ld_wit(p, v);
      s.flag = old >= ominus_cap<V>(gather(p.f + we.x), we.y, p.g.cap);
    }
    __syncthreads();
    if (s.flag) {
      if (threadIdx.x == 0) ++L.witness;
      return false;
    }
  }
  const uint32_t b = __ldg(p.g.off + v), e = __ldg(p.g.off + v + 1);
  if (threadIdx.x == 0) {
    ++L.apps;
    L.edges += e - b;
  }
  V acc = P0 ? TOP : V(0);
  int2 best = make_int2(0, 0);
  bool have = false;
  for (uint32_t i0 = b; i0 < e; i0 += 4 * kBlock) {
    int2 r[4];
    V c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t i = i0 + k * kBlock + threadIdx.x;
      if (i < e) r[k] = ld_rec(p.g, i);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t i = i0 + k * kBlock + threadIdx.x;
      if (i < e) c[k] = ominus_cap<V>(gather(p.f + r[k].x), r[k].y, p.g.cap);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t i = i0 + k * kBlock + threadIdx.x;
      if (i < e) {
        if (P0) {
          if (!have || c[k] < acc) {
            acc = c[k];
            best = r[k];
            have = true;
          }
        } else {
          acc = c[k] > acc ? c[k] : acc;
        }
      }
    }
    const bool done = P0 ? acc == V(0) : acc == TOP;
    if (__syncthreads_or(done)) break;
  }
  // block reduction (value, then the witness record of a minimising lane)
  V wv = P0 ? warp_min(acc) : warp_max(acc);
  int2 wr = best;
  if (P0) {
    const uint32_t m = __ballot_sync(0xffffffffu, have && acc == wv);
    const int src = m ? __ffs(m) - 1 : 0;
    wr.x = __shfl_sync(0xffffffffu, best.x, src);
    wr.y = __shfl_sync(0xffffffffu, best.y, src);
    if (!m) wv = TOP;
  }
  __syncthreads();
  if (lane == 0) {
    s.val[warp] = wv;
    s.rec[warp] = wr;
  }
  __syncthreads();
  bool raised = false;
  if (threadIdx.x == 0) {
    V res = s.val[0];
    int2 rec = s.rec[0];
    for (int w = 1; w < kWarps; ++w) {
      if (P0 ? s.val[w] < res : s.val[w] > res) {
        res = s.val[w];
        rec = s.rec[w];
      }
    }
    if (P0) st_wit(p, v, rec);
    if (store_raise<V, INPLACE>(p, v, res, old)) {
      ++L.lifts;
      raised = true;
    }
    s.flag = raised;
  }
  __syncthreads();
  raised = s.flag;
  __syncthreads();
  return raised;
}

// Warp-uniform dynamic claims of medium rows, kClaim consecutive items per
// atomic so hundreds of thousands of R-MAT rows do not serialise on one
// cursor.  Returns false when the items are exhausted.
constexpr uint32_t kClaim = 8;
struct WarpClaim {
  uint32_t next = 0, end = 0;
};
__device__ __forceinline__ bool warp_claim(unsigned int* cursor, uint32_t count, WarpClaim& c,
                                           uint32_t& item) {
  if (c.next >= c.end) {
    uint32_t base = 0;
    if (lane_id() == 0) base = atomicAdd(cursor, kClaim);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= count) return false;
    c.next = base;
    c.end = base + kClaim < count ? base + kClaim : count;
  }
  item = c.next++;
  return true;
}


// Player-1 light rows of a dense round, TMA-staged.  A warp owns aligned
// 32-vertex tiles; the tile's contiguous span of edge records is brought
// into the warp's shared-memory stage by one bulk copy (cp.async.bulk,
// mbarrier completion) issued one tile ahead, so the HBM stream overlaps the
// gathers of the current tile and never goes through the per-thread LSU
// path.  Tiles whose vertices are all at top are skipped without a copy.
// Each lane then lifts its own row from shared memory (reads rotated by
// lane, so a half-warp hits distinct banks).
constexpr uint32_t kStageRecs = kStageBytes / sizeof(ERec);  // 4 KB per warp stage
// bulk copies move 16-byte multiples from 16-byte aligned addresses
constexpr uint32_t kRecAlign = 16 / sizeof(ERec);

// Per-warp stage barriers live for the whole persistent launch: initialised
// once by k_solve, their phase parity carried across rounds.
__shared__ __align__(8) uint64_t g_tma_bar[kWarps][kStages];
__shared__ uint32_t g_tma_parity[kWarps];

__device__ __forceinline__ void tma_init_barriers() {
  if (lane_id() == 0) {
    const uint32_t warp = threadIdx.x >> 5;
    for (uint32_t s = 0; s < kStages; ++s) mbar_init(&g_tma_bar[warp][s], 1);
    g_tma_parity[warp] = 0;
    mbar_init_fence();
  }
  __syncthreads();
}

// The TMA tile pipeline over the aligned 32-vertex words (tiles) of the
// vertex ranges [lo0, hi0) and [lo1, hi1) (either may be empty): warps claim
// kTileClaim consecutive tiles at a time from `cursor` (a zeroed per-phase
// counter), so a slow SM or a tile of long rows does not hold up the phase.
// Per tile, `load(v, aux)` issues the loads of vertex v's state into a
// per-lane value carried to the row step, `test(v, aux)` says whether v's
// row must be read (only asked for the set bits of the tile's word of
// `mask`, when given), `row(v, rec, len, b, aux)` processes a row held in
// shared memory, `fallback(v, aux)` a row whose tile span does not fit a
// stage (direct loads).  Both return "raised"; raised vertices are
// published in `chg` with one atomicOr per word.
// Per warp, while tile i is processed from its stage, the bulk copies of
// tiles i+1 .. i+kStages-1 are in flight and the vertex state and row
// offsets of the tile after them are loading: the HBM latency of a copy
// (~1-2 us) is covered by the work of the tiles ahead of it.
#ifndef EGS_TILE_CLAIM
#define EGS_TILE_CLAIM 4
#endif
constexpr uint32_t kTileClaim = EGS_TILE_CLAIM;

struct NoAfter {
  __device__ void operator()(uint32_t, bool) const {}
};

template <class V, class Load, class Test, class Row, class Fallback, class After = NoAfter>
__device__ __forceinline__ void tma_tiles(const SolveParams<V>& p, bool staged, uint32_t lo0,
                                          uint32_t hi0, uint32_t lo1, uint32_t hi1,
                                          unsigned int* cursor, const uint32_t* mask,
                                          uint32_t* chg, Local& L, Load load, Test test,
                                          Row row, Fallback fallback, After after = After{}) {
  extern __shared__ __align__(128) ERec dsm[];
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  ERec* stage_base = dsm + (size_t)warp * kStages * kStageRecs;
  uint64_t* s_bar = g_tma_bar[warp];
  const uint32_t T0 = hi0 > lo0 ? ((hi0 + 31) >> 5) - (lo0 >> 5) : 0u;
  const uint32_t T1 = hi1 > lo1 ? ((hi1 + 31) >> 5) - (lo1 >> 5) : 0u;
  const uint32_t T = T0 + T1;
  uint32_t c_next = 0, c_end = 0;  // this warp's current claim (warp-uniform)
  auto claim = [&]() -> uint32_t {
    if (c_next >= c_end) {
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(cursor, kTileClaim);
      base = __shfl_sync(0xffffffffu, base, 0);
      c_next = base;
      c_end = base + kTileClaim < T ? base + kTileClaim : T;
      if (base >= T) return 0xFFFFFFFFu;
    }
    return c_next++;
  };

  if (!staged) {  // direct: every needed row through `fallback` (plain loads)
    for (;;) {
      const uint32_t i = claim();
      if (i >= T) break;
      const bool second = i >= T0;
      const uint32_t w = second ? (lo1 >> 5) + (i - T0) : (lo0 >> 5) + i;
      const uint32_t v = (w << 5) + lane;
      const bool in = v >= (second ? lo1 : lo0) && v < (second ? hi1 : hi0);
      const uint32_t mw = mask ? ldcg(mask + w) : ~0u;
      V aux = V(0);
      bool work = false;
      if (in && ((mw >> lane) & 1u)) {
        load(v, aux);
        work = test(v, aux);
      }
      if (in && !work) ++L.visits;
      const bool ch = work && fallback(v, aux);
      const uint32_t m = __ballot_sync(0xffffffffu, ch);
      if (m && lane == 0) bits_or(p, chg + w, m);
      L.phase_count += ch;
      after(v, ch);  // warp-uniform
    }
    return;
  }

  struct Tile {
    V aux;
    uint32_t w, lo, hi, b, e, base, mask;
    bool valid, in, work, any, staged;
  };
  // step 1: claim a tile and issue the loads of its vertex state and offsets
  auto fetch = [&](Tile& t) {
    const uint32_t i = claim();
    t.valid = i < T;
    t.in = false;
    t.aux = V(0);
    t.b = t.e = 0;
    if (!t.valid) return;
    const bool second = i >= T0;
    t.w = second ? (lo1 >> 5) + (i - T0) : (lo0 >> 5) + i;
    t.lo = second ? lo1 : lo0;
    t.hi = second ? hi1 : hi0;
    const uint32_t v = (t.w << 5) + lane;
    t.in = v >= t.lo && v < t.hi;
    t.mask = mask ? ldcg(mask + t.w) : ~0u;
    if (t.in) {
      load(v, t.aux);
      t.b = __ldg(p.g.off + v);
      t.e = __ldg(p.g.off + v + 1);
    }
  };
  // step 2: if any row of the tile is needed, start the bulk copy of the
  // tile's edge span into stage `s`
  auto prepare = [&](uint32_t s, Tile& t) {
    const uint32_t v = (t.w << 5) + lane;
    t.work = t.in && ((t.mask >> lane) & 1u) && test(v, t.aux);
    t.any = __any_sync(0xffffffffu, t.work);
    t.staged = false;
    if (!t.any) return;
    const uint32_t first = max(t.w << 5, t.lo), last = min((t.w << 5) + 32, t.hi);
    const uint32_t span_lo = __shfl_sync(0xffffffffu, t.b, first - (t.w << 5));
    const uint32_t span_hi = __shfl_sync(0xffffffffu, t.e, last - 1 - (t.w << 5));
    const uint32_t a_lo = span_lo & ~(kRecAlign - 1u);  // 16 B aligned
    const uint32_t a_hi = (span_hi + kRecAlign - 1u) & ~(kRecAlign - 1u);
    t.base = a_lo;
    if (a_hi - a_lo <= kStageRecs) {
      t.staged = true;
      if (lane == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&s_bar[s], (a_hi - a_lo) * (uint32_t)sizeof(ERec));
        bulk_g2s(stage_base + s * kStageRecs, erecs(p.g) + a_lo,
                 (a_hi - a_lo) * (uint32_t)sizeof(ERec), &s_bar[s]);
      }
    }
  };
  auto compute = [&](uint32_t s, const Tile& t, uint32_t& parity) {
    if (t.in && !t.work) ++L.visits;  // e.g. a top vertex: one load, no lift
    if (!t.any) return;
    const uint32_t v = (t.w << 5) + lane;
    bool ch = false;
    if (t.staged) {
      mbar_wait(&s_bar[s], (parity >> s) & 1u);
      parity ^= 1u << s;
      if (t.work) ch = row(v, stage_base + s * kStageRecs + (t.b - t.base), t.e - t.b, t.b, t.aux);
    } else if (t.work) {
      ch = fallback(v, t.aux);
    }
    const uint32_t m = __ballot_sync(0xffffffffu, ch);
    if (m && lane == 0) bits_or(p, chg + t.w, m);
    L.phase_count += ch;
    after(v, ch);  // warp-uniform
  };

  // tile i is processed from slot i % kStages while the copies of tiles
  // i+1 .. i+D are in flight and tile i+D+1 is loading its offsets
  constexpr uint32_t D = kStages - 1;
  uint32_t parity = g_tma_parity[warp];
  Tile t[D + 2];
#pragma unroll
  for (uint32_t k = 0; k <= D; ++k) fetch(t[k]);
#pragma unroll
  for (uint32_t k = 0; k < D; ++k)
    if (t[k].valid) prepare(k, t[k]);
  uint32_t s = 0;
  while (t[0].valid) {
    __syncwarp();  // slot (s + D) % kStages was last read by this warp's previous tile
    if (t[D].valid) prepare(s == 0 ? D : s - 1, t[D]);
    fetch(t[D + 1]);
    compute(s, t[0], parity);
#pragma unroll
    for (uint32_t k = 0; k <= D; ++k) t[k] = t[k + 1];
    s = s == D ? 0 : s + 1;
  }
  __syncwarp();
  if (lane == 0) g_tma_parity[warp] = parity;
  __syncwarp();  // every lane sees the new parity before the warp's next pipeline
}

// Rows of a tile sit back to back in the stage; a lane starts its row at a
// rotation chosen so the lanes of one shared-memory wavefront (32 lanes of
// 4-byte records, 16 of 8-byte ones) hit distinct banks when the rows have
// equal length (exact for lengths dividing 32 / 16).
__device__ __forceinline__ uint32_t row_rot(uint32_t len) {
  constexpr uint32_t G = 128 / sizeof(ERec);  // lanes per wavefront
  return (((lane_id() % G) * len) / G) % len;
}

// f(j) for every record j of a light row, in the rotated order.  A
// power-of-two row of at least kChunk records takes j = k ^ rot instead of
// (k + rot) mod len: the same banks (rot < len spreads the lanes that share a
// start bank), one op per record instead of a clamp and a wrap.  Rows
// shorter than a chunk repeat their last record (idempotent for min / max).
template <class F>
__device__ __forceinline__ void row_edges(uint32_t len, uint32_t rot, F&& f) {
  if ((len & (len - 1)) == 0 && len >= (uint32_t)kChunk) {
    for (uint32_t k0 = 0; k0 < len; k0 += kChunk) {
#pragma unroll
      for (int k = 0; k < kChunk; ++k) f((k0 + k) ^ rot);
    }
  } else {
    for (uint32_t k0 = 0; k0 < len; k0 += kChunk) {
#pragma unroll
      for (int k = 0; k < kChunk; ++k) {
        uint32_t j = min(k0 + k, len - 1) + rot;
        f(j >= len ? j - len : j);
      }
    }
  }
}

// Player-1 light rows of a dense round through the tile pipeline: tiles of
// all-top vertices are skipped without a copy; each lane lifts its own row
// from shared memory (reads rotated by lane so a half-warp hits distinct
// banks), 8 gathers in flight.
// Player-1 light rows of the dense round right after a certificate apply:
// only the vertices the apply listed as still below top (most player-1
// vertices were just certified), one per lane, whole warps busy.
template <class V>
__device__ __noinline__ void dense_light_p1_listed(const SolveParams<V>& p, const uint32_t* list,
                                                   uint32_t count, uint32_t* chg,
                                                   unsigned int* sum_dst) {
  Local L;
  const uint32_t nthreads = gridDim.x * kBlock;
  for (uint32_t i0 = blockIdx.x * kBlock + (threadIdx.x & ~31u); i0 < count; i0 += nthreads) {
    const uint32_t i = i0 + lane_id();
    uint32_t v = 0;
    bool ch = false;
    if (i < count) {
      v = ldcg(list + i);
      ch = lift_thread<V, false>(p, v, L);
    }
    if (ch) {
      set_bit(p, chg, v);
      ++L.phase_count;
    }
  }
  block_flush(L, sum_dst);
}

template <class V, bool INPLACE = false>
__device__ __noinline__ void dense_light_p1(const SolveParams<V>& p, uint32_t lo, uint32_t hi,
                                            unsigned int* cursor, uint32_t* chg,
                                            unsigned int* sum_dst) {
  constexpr V TOP = Top<V>::v;
  Local L;
  auto load = [&](uint32_t v, V& old) { old = ldcg(p.f + v); };
  auto test = [&](uint32_t, V old) { return old != TOP; };
  auto row = [&](uint32_t v, const ERec* rec, uint32_t len, uint32_t, V old) {
    ++L.visits;
    ++L.apps;
    L.edges += len;
    const uint32_t rot = row_rot(len);  // light rows are non-empty
    V acc = 0;
    for (uint32_t k0 = 0; k0 < len; k0 += kChunk) {
      int2 r[kChunk];
#pragma unroll
      for (int k = 0; k < kChunk; ++k) {
        uint32_t j = min(k0 + k, len - 1) + rot;  // clamp (duplicate), rotate banks
        j = j >= len ? j - len : j;
        r[k] = dec(p.g, rec[j]);
      }
      V c[kChunk];
#pragma unroll
      for (int k = 0; k < kChunk; ++k) c[k] = gather(p.f + r[k].x);
#pragma unroll
      for (int k = 0; k < kChunk; ++k) {
        const V x = ominus_cap<V>(c[k], r[k].y, p.g.cap);
        acc = x > acc ? x : acc;
      }
      if (acc == TOP) break;
    }
    if (store_raise<V, INPLACE>(p, v, acc, old)) {
      ++L.lifts;
      return true;
    }
    return false;
  };
  auto fallback = [&](uint32_t v, V) { return lift_thread<V, false, INPLACE>(p, v, L); };
  tma_tiles<V>(p, (p.use_tma & kTmaLift) != 0, lo, hi, 0u, 0u, cursor, nullptr, chg, L, load,
               test, row, fallback);
  block_flush(L, sum_dst);
}

// Player-0 light rows of a dense round.  Almost every player-0 lift is
// settled by its witness edge, so the cost is one dependent gather per
// vertex; a lane takes four vertices (one per 32-vertex word of a 128-vertex
// group) so four witness gathers are in flight per thread.  Vertices whose
// witness is violated are compacted into a per-warp shared-memory queue and
// re-lifted 32 at a time, one row per lane, so a few violated rows never
// serialise a warp.
#ifndef EGS_P0_UNROLL
#define EGS_P0_UNROLL 4
#endif
constexpr int kP0Unroll = EGS_P0_UNROLL;
// the per-warp queue of violated rows (one allocation for both instantiations)
__shared__ uint32_t g_p0_queue[kWarps][32 * kP0Unroll + 32];

template <class V, bool INPLACE = false>
__device__ __noinline__ void dense_light_p0(const SolveParams<V>& p, uint32_t lo, uint32_t hi,
                                            uint32_t* chg, unsigned int* sum_dst) {
  constexpr V TOP = Top<V>::v;
  constexpr int U = kP0Unroll;
  Local L;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  uint32_t* q = g_p0_queue[warp];
  uint32_t qn = 0;  // warp-uniform queue length
  auto drain = [&](uint32_t keep) {
    while (qn > keep) {
      const uint32_t take = qn - keep < 32u ? qn - keep : 32u;
      const uint32_t base = qn - take;
      __syncwarp();
      bool ch = false;
      uint32_t v = 0;
      if (lane < take) {
        v = q[base + lane];
        ch = lift_thread<V, true, INPLACE>(p, v, L);
      }
      if (ch) set_bit(p, chg, v);
      L.phase_count += ch;
      qn = base;
      __syncwarp();
    }
  };
  const uint32_t nwarps = gridDim.x * kWarps;
  const uint32_t gw = blockIdx.x * kWarps + warp;
  const uint32_t w0 = lo >> 5, w1 = (hi + 31) >> 5;
  for (uint32_t wb = w0 + gw * U; wb < w1; wb += nwarps * U) {
    V old[U], cw[U];
    int2 we[U];
    bool in[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint32_t v = ((wb + k) << 5) + lane;
      in[k] = wb + k < w1 && v >= lo && v < hi;
      old[k] = in[k] ? ldcg(p.f + v) : TOP;
      we[k] = in[k] ? ld_wit(p, v) : make_int2(0, 0);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) cw[k] = old[k] != TOP ? gather(p.f + we[k].x) : TOP;
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint32_t v = ((wb + k) << 5) + lane;
      bool viol = false;
      if (in[k]) {
        ++L.visits;
        if (old[k] != TOP) {
          viol = old[k] < ominus_cap<V>(cw[k], we[k].y, p.g.cap);
          L.witness += !viol;
        }
      }
      const uint32_t m = __ballot_sync(0xffffffffu, viol);
      if (viol) {
        --L.visits;  // lift_thread counts its own visit
        q[qn + __popc(m & lanemask_lt())] = v;
      }
      qn += __popc(m);
    }
    drain(31);  // keep fewer than a warp's worth queued
  }
  drain(0);
  block_flush(L, sum_dst);
}

// Activation (solver_par.cpp:402-410): every non-top predecessor of a vertex
// marked in `chg` enters frontier buffer `nb` once (bitmap dedup), sorted
// into its size-class sublist; the warp expands CSC columns as one stream.
// Columns longer than kLongCol (the in-hubs of a power-law arena) are not
// expanded by one warp: they are queued in p.longcol (count in qlong) for
// phase_activate_long, which spreads their chunks over the whole grid.

// Frontier appends are buffered per warp in shared memory (the TMA stage
// area, idle during activation) and published up to kAppendCap entries per
// atomicAdd, so a large frontier does not serialise on the three list
// counters.  Warp-uniform.
constexpr uint32_t kAppendCap = 512;  // entries per class per warp (3 * 2 KB)

struct WarpLists {
  uint32_t* buf[3];
  uint32_t cnt[3];
  uint32_t cap;  // entries per class buffer
};

// A frontier being produced: its three class sublists, their counters and
// its membership (dedup) bitmap.  Frontiers are numbered tokens: token k
// lives in list buffer k & 1 with bitmap p.frb[k & 1] and counters
// fr_cnt[k % 3], so the producer of token k can zero the counters of token
// k + 1 while token k - 1 is still being read (k_solve main loop).
struct Frontier {
  uint32_t* list[3];
  unsigned int* cnt;
  uint32_t* frb;
};

__device__ __forceinline__ WarpLists warp_lists() {
  extern __shared__ __align__(128) ERec dsm[];
  uint32_t* base = reinterpret_cast<uint32_t*>(dsm) +
                   (size_t)(threadIdx.x >> 5) * (kStages * kStageBytes / 4);
  WarpLists q;
  for (int c = 0; c < 3; ++c) {
    q.buf[c] = base + c * kAppendCap;
    q.cnt[c] = 0;
  }
  q.cap = kAppendCap;
  return q;
}

// Small per-warp buffers in static shared memory, for phases whose dynamic
// shared memory holds TMA stages (the certificate pass's re-check pushes).
constexpr uint32_t kSmallAppendCap = 64;
__device__ __forceinline__ WarpLists warp_lists_small() {
  __shared__ uint32_t s_lists[kWarps][3][kSmallAppendCap];
  WarpLists q;
  for (int c = 0; c < 3; ++c) {
    q.buf[c] = s_lists[threadIdx.x >> 5][c];
    q.cnt[c] = 0;
  }
  q.cap = kSmallAppendCap;
  return q;
}

__device__ __forceinline__ void lists_flush(WarpLists& q, int c, uint32_t* list,
                                            unsigned int* count) {
  __syncwarp();
  const uint32_t k = q.cnt[c];
  if (k == 0) return;
  uint32_t base = 0;
  if (lane_id() == 0) base = atomicAdd(count, k);
  base = __shfl_sync(0xffffffffu, base, 0);
  for (uint32_t i = lane_id(); i < k; i += 32) list[base + i] = q.buf[c][i];
  q.cnt[c] = 0;
  __syncwarp();
}

__device__ __forceinline__ void lists_append(WarpLists& q, bool pred, int c, uint32_t v,
                                             uint32_t* const* lists, unsigned int* counts) {
#pragma unroll
  for (int cc = 0; cc < 3; ++cc) {
    const bool mine = pred && c == cc;
    const uint32_t m = __ballot_sync(0xffffffffu, mine);
    if (!m) continue;
    if (mine) q.buf[cc][q.cnt[cc] + __popc(m & lanemask_lt())] = v;
    q.cnt[cc] += __popc(m);
    if (q.cnt[cc] + 32 > q.cap) lists_flush(q, cc, lists[cc], counts + cc);
  }
}

template <class V>
__device__ __forceinline__ void activate_pred(const SolveParams<V>& p, bool valid, uint32_t idx,
                                              WarpLists& q, const Frontier& t, Local& L,
                                              bool pushing = false, bool cert = false) {
  const Graph& g = p.g;
  bool add = false;
  uint32_t u = 0;
  int c = 0;
  if (valid) {
    if (!cert) ++L.act;
    u = __ldg(g.csrc + idx);
    const uint32_t bit = 1u << (u & 31u);
    // a plain read first: predecessors shared by many changed vertices (the
    // in-hubs' neighbours) are already marked and skip the atomic.  The
    // certificate's re-check queue takes the owned candidates instead of the
    // non-top vertices.
    const bool want = cert ? owned(p, u) && ((ldcg(p.cand + (u >> 5)) >> (u & 31u)) & 1u)
                           : gather(p.f + u) != Top<V>::v;
    if (!(ldcg(t.frb + (u >> 5)) & bit) && want) {
      add = !(atomicOr(t.frb + (u >> 5), bit) & bit);
      c = size_class(g, u);
    }
  }
  lists_append(q, add, c, u, t.list, t.cnt);
  if (pushing)
    L.pushed += add;
  else
    L.phase_count += add;
}

// activate_pred for U predecessor slots per lane: the source loads, then the
// membership tests (top / candidate gathers and dedup words), then the
// dedup atomics of all U are issued before any result is used.
#ifndef EGS_ACT_UNROLL
#define EGS_ACT_UNROLL 2
#endif
constexpr int kActUnroll = EGS_ACT_UNROLL;

template <class V, int U>
__device__ __forceinline__ void activate_preds(const SolveParams<V>& p, const bool (&valid)[U],
                                               const uint32_t (&idx)[U], WarpLists& q,
                                               const Frontier& t, Local& L, bool pushing,
                                               bool cert) {
  const Graph& g = p.g;
  uint32_t u[U], fr[U];
  bool want[U], add[U];
#pragma unroll
  for (int k = 0; k < U; ++k) u[k] = valid[k] ? __ldg(g.csrc + idx[k]) : 0u;
#pragma unroll
  for (int k = 0; k < U; ++k) {
    want[k] = false;
    fr[k] = ~0u;
    if (valid[k]) {
      want[k] = cert ? owned(p, u[k]) && ((ldcg(p.cand + (u[k] >> 5)) >> (u[k] & 31u)) & 1u)
                     : gather(p.f + u[k]) != Top<V>::v;
      fr[k] = ldcg(t.frb + (u[k] >> 5));
    }
  }
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const uint32_t bit = 1u << (u[k] & 31u);
    add[k] = valid[k] && want[k] && !(fr[k] & bit) && !(atomicOr(t.frb + (u[k] >> 5), bit) & bit);
  }
#pragma unroll
  for (int k = 0; k < U; ++k) {
    if (valid[k] && !cert) ++L.act;
    lists_append(q, add[k], add[k] ? size_class(g, u[k]) : 0, u[k], t.list, t.cnt);
    if (pushing)
      L.pushed += add[k];
    else
      L.phase_count += add[k];
  }
}

// the predecessors of CSC range [b, e) of each lane, expanded by the warp
template <class V>
__device__ __forceinline__ void expand_preds(const SolveParams<V>& p, uint32_t b, uint32_t e,
                                             WarpLists& q, const Frontier& t, Local& L,
                                             bool pushing, bool cert) {
  if (kActUnroll > 1) {
    warp_expand_n<kActUnroll>(b, e, [&](const bool(&valid)[kActUnroll],
                                        const uint32_t(&idx)[kActUnroll]) {
      activate_preds<V, kActUnroll>(p, valid, idx, q, t, L, pushing, cert);
    });
  } else {
    warp_expand(b, e, [&](bool valid, uint32_t idx, uint32_t) {
      activate_pred<V>(p, valid, idx, q, t, L, pushing, cert);
    });
  }
}

// Certificate passes push the candidate predecessors of each removed vertex
// into the next pass's re-check queue `t` (dedup bitmap t.frb).  Warp-uniform.
template <class V>
__device__ __forceinline__ void push_cert_preds(const SolveParams<V>& p, bool removed, uint32_t v,
                                                WarpLists& q, const Frontier& t, Local& L) {
  if (!t.cnt || !__any_sync(0xffffffffu, removed)) return;
  uint32_t b = 0, e = 0;
  if (removed) {
    b = __ldg(p.g.coff + v);
    e = __ldg(p.g.coff + v + 1);
  }
  expand_preds<V>(p, b, e, q, t, L, true, true);
}

// Push activation of a sparse round: the predecessors of the vertices of the
// lanes with `raised` enter frontier t right away (one CSC column per such
// lane, expanded by the whole warp; columns longer than kLongCol are queued
// for phase_activate_long).  Warp-uniform.
template <class V>
__device__ __forceinline__ void push_preds(const SolveParams<V>& p, bool raised, uint32_t v,
                                           WarpLists& q, const Frontier& t,
                                           unsigned int* qlong, Local& L) {
  // several ranks: the replicated changed bitmap feeds phase_activate
  // instead (a rank cannot push the predecessors of its peers' raises)
  if (p.world > 1 || !__any_sync(0xffffffffu, raised)) return;
  uint32_t b = 0, e = 0;
  if (raised) {
    b = __ldg(p.g.coff + v);
    e = __ldg(p.g.coff + v + 1);
    if (e - b > kLongCol) {
      const uint32_t k = atomicAdd(qlong, 1u);
      p.longcol[2 * k] = v;
      p.longcol[2 * k + 1] = 0u;
      e = b;
    }
  }
  expand_preds<V>(p, b, e, q, t, L, true, false);
}

// Light rows of a sparse frontier list, one thread each, lifted in place;
// raised vertices push their predecessors into frontier `nxt`.
template <class V>
__device__ __noinline__ void sparse_light(const SolveParams<V>& p, const uint32_t* list,
                                          uint32_t count, uint32_t* chg,
                                          unsigned int* sum_dst, Frontier nxt,
                                          unsigned int* qlong, unsigned int* act_dst) {
  Local L;
  WarpLists q = warp_lists();
  const uint32_t nthreads = gridDim.x * kBlock;
  const uint32_t base = blockIdx.x * kBlock + (threadIdx.x & ~31u);
  for (uint32_t i0 = base; i0 < count; i0 += nthreads) {  // warp-uniform loop
    const uint32_t i = i0 + lane_id();
    uint32_t v = 0;
    bool ch = false;
    if (i < count) {
      v = ldcg(list + i);
      ch = v < p.g.rb[kP1L] ? lift_thread<V, true, true>(p, v, L)
                            : lift_thread<V, false, true>(p, v, L);
    }
    if (ch) {
      set_bit(p, chg, v);
      ++L.phase_count;
    }
    push_preds<V>(p, ch, v, q, nxt, qlong, L);
  }
  for (int c = 0; c < 3; ++c) lists_flush(q, c, nxt.list[c], nxt.cnt + c);
  block_flush(L, sum_dst, act_dst);
}

// Medium rows: warps claim rows from a per-phase cursor.  `items(i)` maps a
// claim index to a vertex.
// With `push` (sparse rounds) rows are lifted in place and a raised row
// pushes its predecessors into frontier `nxt`.
template <class V, class Items>
__device__ __noinline__ void warp_rows(const SolveParams<V>& p, uint32_t count,
                                          unsigned int* cursor, Items items,
                                          uint32_t* chg, unsigned int* sum_dst,
                                          bool push = false, Frontier nxt = Frontier{},
                                          unsigned int* qlong = nullptr,
                                          unsigned int* act_dst = nullptr,
                                          bool inplace = false) {
  Local L;
  WarpLists q = warp_lists();
  WarpClaim wc;
  uint32_t i;
  while (warp_claim(cursor, count, wc, i)) {
    const uint32_t v = items(i);
    if (!owned(p, v)) continue;
    const bool p0 = v < p.g.rb[kP1L];
    bool ch;
    if (push || inplace)
      ch = p0 ? lift_warp<V, true, true>(p, v, L) : lift_warp<V, false, true>(p, v, L);
    else
      ch = p0 ? lift_warp<V, true>(p, v, L) : lift_warp<V, false>(p, v, L);
    if (ch && lane_id() == 0) {
      set_bit(p, chg, v);
      ++L.phase_count;
    }
    if (push) push_preds<V>(p, ch && lane_id() == 0, v, q, nxt, qlong, L);
  }
  if (push)
    for (int c = 0; c < 3; ++c) lists_flush(q, c, nxt.list[c], nxt.cnt + c);
  block_flush(L, sum_dst, act_dst);
}

template <class V, class Items>
__device__ __noinline__ void block_rows(const SolveParams<V>& p, uint32_t count,
                                           unsigned int* cursor, Items items,
                                           uint32_t* chg, unsigned int* sum_dst,
                                           bool push = false, Frontier nxt = Frontier{},
                                           unsigned int* qlong = nullptr,
                                           unsigned int* act_dst = nullptr,
                                           bool inplace = false) {
  __shared__ BlockScratch<V> s;
  Local L;
  WarpLists q = warp_lists();
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s.item = atomicAdd(cursor, 1u);
    __syncthreads();
    const uint32_t i = s.item;
    if (i >= count) break;
    const uint32_t v = items(i);
    if (!owned(p, v)) continue;
    const bool p0 = v < p.g.rb[kP1L];
    bool ch;
    if (push || inplace)
      ch = p0 ? lift_block<V, true, true>(p, v, L, s) : lift_block<V, false, true>(p, v, L, s);
    else
      ch = p0 ? lift_block<V, true>(p, v, L, s) : lift_block<V, false>(p, v, L, s);
    if (ch && threadIdx.x == 0) {
      set_bit(p, chg, v);
      ++L.phase_count;
    }
    if (push && threadIdx.x < 32)  // warp 0 expands the raised hub's column
      push_preds<V>(p, ch && threadIdx.x == 0, v, q, nxt, qlong, L);
  }
  __syncthreads();
  if (push && threadIdx.x < 32)
    for (int c = 0; c < 3; ++c) lists_flush(q, c, nxt.list[c], nxt.cnt + c);
  block_flush(L, sum_dst, act_dst);
}

// ======================================================= certificate ====
// Losing-region certificate.  A pass keeps candidate v iff
//   player 0: every edge (v,t) is good;  player 1: some edge (v,t) is good,
// good(v,t) = f(t) = top, or t is a candidate and f(v) < f(t) - w(v,t).
// Removal is in place; the greatest fixpoint is reached when a pass removes
// nothing.  Every candidate left is in W1: under the good-edge choices every
// step inside the set changes the energy by w <= f(t) - f(v) - 1, so any
// cycle player 0 can close there is negative.
// Candidates are marked twice: a bit in p.cand (one per vertex, 2 MB at
// C4: tile masks, the sparse passes, apply) and the top bit of their value in
// f (kCand, free because credit_cap < 2^(bits-1) - 1 on the device), so an
// edge test is ONE gather: good(v,t) = f(t) = top, or f(t) carries kCand and
// f(v) < value(t) - w(v,t).  f is not otherwise written during the
// certificate; a removed candidate gets its plain value back, a certified one
// becomes top (which has every bit set), so no mark outlives the attempt.
template <class V>
struct CandFlag {
  static constexpr V v = V(1) << (sizeof(V) * 8 - 1);
};
template <class V>
__device__ __forceinline__ int64_t cand_value(V x) {
  return static_cast<int64_t>(x & ~CandFlag<V>::v);
}
template <class V>
__device__ __forceinline__ bool good_target(int64_t fv, V ft, int w) {
  return ft == Top<V>::v || ((ft & CandFlag<V>::v) && fv < cand_value<V>(ft) - w);
}
template <class V>
__device__ __forceinline__ bool cand_bit(const SolveParams<V>& p, uint32_t v) {
  return (ldcg(p.cand + (v >> 5)) >> (v & 31u)) & 1u;
}
// removal of candidate v with value fv: clear its bit and its mark in f
template <class V>
__device__ __forceinline__ void cand_clear(const SolveParams<V>& p, uint32_t v, int64_t fv) {
  atomicAnd(p.cand + (v >> 5), ~(1u << (v & 31u)));
  f_put<V>(p, v, static_cast<V>(fv));
}
template <class V>
__device__ __forceinline__ bool good_edge(const SolveParams<V>& p, int64_t fv, int2 r) {
  return good_target<V>(fv, gather(p.f + r.x), r.y);
}

#ifndef EGS_CERT_CHUNK
#define EGS_CERT_CHUNK 4
#endif
#ifndef EGS_DENSE_COMMIT_DIV
#define EGS_DENSE_COMMIT_DIV 8
#endif
// a commit loads all staged slots when at least n / kDenseCommitDiv were raised
// (0: never)
constexpr uint64_t kDenseCommitDiv = EGS_DENSE_COMMIT_DIV;
#ifndef EGS_PACKED_WITNESS_KEY
#define EGS_PACKED_WITNESS_KEY 1
#endif
// round 1's player-0 witness as one packed min per edge (4-byte records with
// tbits >= 5, so |w| < 2^26: round1_light)
constexpr bool kPackedWitnessKey = EGS_PACKED_WITNESS_KEY != 0 && EGS_EDGE_BYTES == 4;
constexpr int kCertChunk = EGS_CERT_CHUNK;  // edges tested per step (early exit between)
#ifndef EGS_CERT_CHUNK_P0
#define EGS_CERT_CHUNK_P0 8
#endif
constexpr int kCertChunkP0 = EGS_CERT_CHUNK_P0;  // player-0 rows in the TMA pass

template <class V, bool P0>
__device__ __forceinline__ bool cert_keep_thread(const SolveParams<V>& p,
                                                 uint32_t v, int64_t fv, Local& L) {
  const uint32_t b = __ldg(p.g.off + v), e = __ldg(p.g.off + v + 1);
  for (uint32_t i = b; i < e; i += kCertChunk) {
    int2 r[kCertChunk];
#pragma unroll
    for (int k = 0; k < kCertChunk; ++k) r[k] = ld_rec(p.g, min(i + k, e - 1));
    V c[kCertChunk];
#pragma unroll
    for (int k = 0; k < kCertChunk; ++k) c[k] = gather(p.f + r[k].x);
    bool all = true, any = false;
#pragma unroll
    for (int k = 0; k < kCertChunk; ++k) {
      const bool g = good_target<V>(fv, c[k], r[k].y);
      all &= g;
      any |= g;
    }
    L.cert_edges += min((uint32_t)kCertChunk, e - i);
    if (P0 && !all) return false;
    if (!P0 && any) return true;
  }
  return P0;
}

template <class V, bool P0>
__device__ __forceinline__ bool cert_keep_warp(const SolveParams<V>& p, uint32_t v,
                                               int64_t fv, Local& L) {
  const uint32_t b = __ldg(p.g.off + v), e = __ldg(p.g.off + v + 1);
  for (uint32_t i = b + lane_id(); i - lane_id() < e; i += 32) {
    bool g = P0;
    if (i < e) {
      ++L.cert_edges;
      g = good_edge<V>(p, fv, ld_rec(p.g, i));
    }
    if (P0 && !__all_sync(0xffffffffu, g)) return false;
    if (!P0 && __any_sync(0xffffffffu, g)) return true;
  }
  return P0;
}

template <class V, bool P0>
__device__ __forceinline__ bool cert_keep_block(const SolveParams<V>& p, uint32_t v,
                                                int64_t fv, Local& L) {
  const uint32_t b = __ldg(p.g.off + v), e = __ldg(p.g.off + v + 1);
  for (uint32_t i0 = b; i0 < e; i0 += kBlock) {
    const uint32_t i = i0 + threadIdx.x;
    bool g = P0;
    if (i < e) {
      ++L.cert_edges;
      g = good_edge<V>(p, fv, ld_rec(p.g, i));
    }
    if (P0 && !__syncthreads_and(g)) return false;
    if (!P0 && __syncthreads_or(g)) return true;
  }
  return P0;
}

// ============================================================ phases ====
// Each phase is a separate non-inlined function so it gets its own register
// allocation; the kernel body only keeps the (grid-uniform) loop state.
// Every phase ends with block_flush; the caller then crosses a grid barrier.

// Round 1 straight from the weights.  With f = 0 everywhere a lift reads no
// measure at all: f(t) ⊖ w = max(0, -w), so delta(0)(v) = max(0, -min_w)
// for player 1 and max(0, -max_w) for player 0.  The vertices it raises are
// exactly the reference's seeds (solver_par.cpp:366-387: player 0 with only
// negative moves, player 1 with some negative move), so this one pass over
// the weights is both the seeding and the first synchronous round of
// solve_frontier / solve_sweep.  The player-0 witness starts at the argmin:
// the first non-negative edge, else the least negative one.
// A round-1 raise.  Round 1 reads the weights only, so with one rank it
// writes f directly (r1_direct: no staging, no commit phase) and, when the
// first certificate attempt follows it (r1_cand), marks the candidates as
// the commit would -- the value's top bit here, the bitmap bit at the
// caller's change ballot.  (A round-1 value is max(0, -w) <= max |w| <=
// credit_cap, never top, so every raised vertex is a candidate.)
template <class V>
__device__ __forceinline__ void r1_store(const SolveParams<V>& p, uint32_t v, V val) {
  if (p.r1_direct)
    stcg(p.f + v, p.r1_cand ? (V)(val | CandFlag<V>::v) : val);
  else
    stcg(p.stage + v, val);
}
// the candidate bits of a word's raised vertices (r1_cand; warp-uniform m)
template <class V>
__device__ __forceinline__ void r1_cand_bits(const SolveParams<V>& p, uint32_t w, uint32_t m) {
  if (p.r1_cand && m && lane_id() == 0) bits_or(p, p.cand + w, m);
}
template <class V>
__device__ __forceinline__ void round1_finish(const SolveParams<V>& p, uint32_t v, bool p0,
                                              int minw, int maxw, uint32_t imax, V& val) {
  val = ominus_cap<V>(V(0), p0 ? maxw : minw, p.g.cap);
  if (p0) stcg(wit_of(p) + v, __ldg(erecs(p.g) + imax));
  if (val > V(0)) r1_store<V>(p, v, val);
}

// light rows: one thread per row over the TMA tile pipeline (the weight scan
// streams the whole edge array once)
template <class V>
__device__ __noinline__ void round1_light(const SolveParams<V>& p, uint32_t lo0, uint32_t hi0,
                                          uint32_t lo1, uint32_t hi1, unsigned int* cursor,
                                          uint32_t* chg, unsigned int* sum_dst) {
  const Graph& g = p.g;
  Local L;
  auto load = [](uint32_t, V&) {};
  auto test = [](uint32_t, V) { return true; };
  auto finish = [&](uint32_t v, bool p0, int minw, int maxw, ERec wrec, uint32_t len) {
    const V val = ominus_cap<V>(V(0), p0 ? maxw : minw, g.cap);
    if (p0) stcg(wit_of(p) + v, wrec);
    ++L.visits;
    ++L.apps;
    L.edges += len;
    if (val > V(0)) {
      r1_store<V>(p, v, val);
      ++L.lifts;
      return true;
    }
    return false;
  };
  // the player-0 witness: an edge of least max(0, -w), preferring a
  // player-0 target (player-1 targets are the ones the certificate sends to
  // top, which would void the witness in the next round)
  auto row = [&](uint32_t v, const ERec* rec, uint32_t len, uint32_t, V) {
    const bool p0 = v < g.rb[kP1L];  // uniform over a tile's working lanes
    const uint32_t rot = row_rot(len);
    if (p0 && kPackedWitnessKey && g.tbits >= 5) {
      // packed records with |w| < 2^26 (tbits >= 5): the key and the index
      // of a light row (< 32) in one word, so the argmin is one min per
      // edge, and the least key's max(0, -w) is max(0, -max w), the value
      uint32_t kb = 0xFFFFFFFFu;
      const uint32_t b1 = g.rb[kP1L];
      row_edges(len, rot, [&](uint32_t j) {
        const int2 r = dec(g, rec[j]);
        kb = min(kb, ((uint32_t)max(0, -r.y) << 6) | ((uint32_t)((uint32_t)r.x >= b1) << 5) | j);
      });
      return finish(v, true, INT32_MAX, -(int)(kb >> 6), rec[kb & 31u], len);
    }
    if (!p0)  // player 1: rows sorted by weight at upload, the least is first
      return finish(v, false, rec_w(g, rec[0]), INT32_MIN, rec[0], len);
    int minw = INT32_MAX, maxw = INT32_MIN;
    uint32_t jbest = 0, kbest = 0xFFFFFFFFu;
    for (uint32_t k0 = 0; k0 < len; k0 += kChunk) {
#pragma unroll
      for (int k = 0; k < kChunk; ++k) {
        uint32_t j = min(k0 + k, len - 1) + rot;
        j = j >= len ? j - len : j;
        const int2 r = dec(g, rec[j]);
        if (p0) {
          maxw = max(maxw, r.y);
          // key = 2 * max(0, -w) + (target is player 1): fits 32 bits
          const uint32_t key = ((r.y >= 0 ? 0u : (uint32_t)(-r.y)) << 1) |
                               (uint32_t)((uint32_t)r.x >= g.rb[kP1L]);
          if (key < kbest) {
            kbest = key;
            jbest = j;
          }
        } else {
          minw = min(minw, r.y);
        }
      }
    }
    return finish(v, p0, minw, maxw, rec[jbest], len);
  };
  auto fallback = [&](uint32_t v, V) {
    const bool p0 = v < g.rb[kP1L];
    const uint32_t b = __ldg(g.off + v), e = __ldg(g.off + v + 1);
    int minw = INT32_MAX, maxw = INT32_MIN;
    uint32_t ibest = b, kbest = 0xFFFFFFFFu;
    for (uint32_t i = b; i < e; i += kChunk) {
      int2 r[kChunk];
#pragma unroll
      for (int k = 0; k < kChunk; ++k) r[k] = ld_rec(g, min(i + k, e - 1));
#pragma unroll
      for (int k = 0; k < kChunk; ++k) {
        minw = min(minw, r[k].y);
        maxw = max(maxw, r[k].y);
        // the witness key of the tile path: least max(0, -w), player-0 target first
        const uint32_t key = ((r[k].y >= 0 ? 0u : (uint32_t)(-r[k].y)) << 1) |
                             (uint32_t)((uint32_t)r[k].x >= g.rb[kP1L]);
        if (key < kbest) {
          kbest = key;
          ibest = min(i + k, e - 1);
        }
      }
    }
    return finish(v, p0, minw, maxw, __ldg(erecs(g) + ibest), e - b);
  };
  auto after = [&](uint32_t v, bool ch) {  // warp-uniform, one tile = one word
    r1_cand_bits<V>(p, v >> 5, __ballot_sync(0xffffffffu, ch));
  };
  tma_tiles<V>(p, (p.use_tma & kTmaRound1) != 0, lo0, hi0, lo1, hi1, cursor, nullptr, chg, L,
               load, test, row, fallback, after);
  block_flush(L, sum_dst);
}

// Player-0 light rows of round 1 with packed records, two bitmap words (64
// rows, two per lane) per TMA copy.  The tile pipeline moves one word per
// copy -- 2 KB for C4's 16-edge rows, half a stage -- with one copy ahead per
// warp, which holds round 1's pure stream to ~2.7 TB/s; a pair fills the
// 4 KB stage and doubles the bytes in flight.  Same result as round1_light's
// packed witness key.  A pair whose span exceeds a stage reads its rows
// directly.  Needs kStages == 2 (the caller checks).
template <class V>
__device__ __noinline__ void round1_p0_pairs(const SolveParams<V>& p, uint32_t lo, uint32_t hi,
                                             unsigned int* cursor, uint32_t* chg,
                                             unsigned int* sum_dst) {
  extern __shared__ __align__(128) ERec dsm[];
  const Graph& g = p.g;
  Local L;
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  ERec* stage_base = dsm + (size_t)warp * kStages * kStageRecs;
  uint64_t* s_bar = g_tma_bar[warp];
  const uint32_t w_lo = lo >> 5, w_hi = hi > lo ? (hi + 31) >> 5 : w_lo;
  const uint32_t U = (w_hi - w_lo + 1) / 2;  // pairs of words
  const uint32_t b1 = g.rb[kP1L];
  uint32_t c_next = 0, c_end = 0;
  auto claim = [&]() -> uint32_t {
    if (c_next >= c_end) {
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(cursor, kTileClaim);
      base = __shfl_sync(0xffffffffu, base, 0);
      c_next = base;
      c_end = base + kTileClaim < U ? base + kTileClaim : U;
      if (base >= U) return 0xFFFFFFFFu;
    }
    return c_next++;
  };
  struct Pair {
    uint32_t w, b[2], e[2], base;
    bool valid, in[2], staged;
  };
  auto fetch = [&](Pair& t) {
    const uint32_t i = claim();
    t.valid = i < U;
    t.in[0] = t.in[1] = false;
    t.b[0] = t.e[0] = t.b[1] = t.e[1] = 0;
    if (!t.valid) return;
    t.w = w_lo + 2 * i;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t v = ((t.w + h) << 5) + lane;
      t.in[h] = v >= lo && v < hi;
      if (t.in[h]) {
        t.b[h] = __ldg(g.off + v);
        t.e[h] = __ldg(g.off + v + 1);
      }
    }
  };
  auto prepare = [&](uint32_t s, Pair& t) {
    const uint32_t v0 = t.w << 5;
    const uint32_t first = max(v0, lo), last = min(v0 + 64, hi) - 1;
    const uint32_t span_lo = __shfl_sync(0xffffffffu, t.b[0], first - v0);
    const uint32_t hi0 = __shfl_sync(0xffffffffu, t.e[0], (last - v0) & 31u);
    const uint32_t hi1 = __shfl_sync(0xffffffffu, t.e[1], (last - v0) & 31u);
    const uint32_t span_hi = last >= v0 + 32 ? hi1 : hi0;
    const uint32_t a_lo = span_lo & ~(kRecAlign - 1u);
    const uint32_t a_hi = (span_hi + kRecAlign - 1u) & ~(kRecAlign - 1u);
    t.base = a_lo;
    t.staged = a_hi - a_lo <= kStageRecs;
    if (t.staged && lane == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&s_bar[s], (a_hi - a_lo) * (uint32_t)sizeof(ERec));
      bulk_g2s(stage_base + s * kStageRecs, erecs(g) + a_lo,
               (a_hi - a_lo) * (uint32_t)sizeof(ERec), &s_bar[s]);
    }
  };
  // packed witness key (round1_light): one min per edge
  auto row = [&](uint32_t v, const ERec* rec, uint32_t len) {
    const uint32_t rot = row_rot(len);
    uint32_t kb = 0xFFFFFFFFu;
    row_edges(len, rot, [&](uint32_t j) {
      const int2 r = dec(g, rec[j]);
      kb = min(kb, ((uint32_t)max(0, -r.y) << 6) | ((uint32_t)((uint32_t)r.x >= b1) << 5) | j);
    });
    const V val = ominus_cap<V>(V(0), -(int)(kb >> 6), g.cap);
    stcg(wit_of(p) + v, rec[kb & 31u]);
    ++L.visits;
    ++L.apps;
    L.edges += len;
    if (val > V(0)) {
      r1_store<V>(p, v, val);
      ++L.lifts;
      return true;
    }
    return false;
  };
  auto direct = [&](uint32_t v, uint32_t b, uint32_t e) {  // the same key from global
    uint32_t kb = 0xFFFFFFFFu;
    for (uint32_t i = b; i < e; ++i) {
      const int2 r = ld_rec(g, i);
      kb = min(kb, ((uint32_t)max(0, -r.y) << 6) | ((uint32_t)((uint32_t)r.x >= b1) << 5) | (i - b));
    }
    const V val = ominus_cap<V>(V(0), -(int)(kb >> 6), g.cap);
    stcg(wit_of(p) + v, __ldg(erecs(g) + b + (kb & 31u)));
    ++L.visits;
    ++L.apps;
    L.edges += e - b;
    if (val > V(0)) {
      r1_store<V>(p, v, val);
      ++L.lifts;
      return true;
    }
    return false;
  };
  auto compute = [&](uint32_t s, const Pair& t, uint32_t& parity) {
    if (t.staged) {
      mbar_wait(&s_bar[s], (parity >> s) & 1u);
      parity ^= 1u << s;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t v = ((t.w + h) << 5) + lane;
      bool ch = false;
      if (t.in[h])
        ch = t.staged ? row(v, stage_base + s * kStageRecs + (t.b[h] - t.base), t.e[h] - t.b[h])
                      : direct(v, t.b[h], t.e[h]);
      const uint32_t m = __ballot_sync(0xffffffffu, ch);
      if (m && lane == 0) bits_or(p, chg + t.w + h, m);
      r1_cand_bits<V>(p, t.w + h, m);
      L.phase_count += ch;
    }
  };
  uint32_t parity = g_tma_parity[warp];
  Pair t0, t1;
  fetch(t0);
  if (t0.valid) prepare(0, t0);
  uint32_t s = 0;
  while (t0.valid) {
    __syncwarp();  // slot s ^ 1 was last read by this warp's previous pair
    fetch(t1);
    if (t1.valid) prepare(s ^ 1u, t1);
    compute(s, t0, parity);
    t0 = t1;
    s ^= 1u;
  }
  __syncwarp();
  if (lane == 0) g_tma_parity[warp] = parity;
  __syncwarp();
  block_flush(L, sum_dst);
}

// medium rows: one warp per row; heavy rows: one CTA per row (dynamic claims)
template <class V>
__device__ __noinline__ void round1_long(const SolveParams<V>& p, uint32_t* chg,
                                         unsigned int* sum_dst, unsigned int* slot_dyn) {
  __shared__ int s_min[kWarps], s_max[kWarps];
  __shared__ uint32_t s_imax[kWarps];
  __shared__ unsigned int s_item;
  const Graph& g = p.g;
  Local L;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  // heavy: the CTA strides the row, block-reduces min / max / argmax
  const uint32_t nH = class_size(g, 2);
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_item = atomicAdd(slot_dyn + 1, 1u);
    __syncthreads();
    const uint32_t it = s_item;
    if (it >= nH) break;
    const uint32_t u = class_item(g, 2, it);
    if (!owned(p, u)) continue;
    const bool p0 = u < g.rb[kP1L];
    const uint32_t b = __ldg(g.off + u), e = __ldg(g.off + u + 1);
    int minw = INT32_MAX, maxw = INT32_MIN;
    uint32_t imax = b;
    for (uint32_t i = b + threadIdx.x; i < e; i += kBlock) {
      const int w = rec_w(g, __ldcs(erecs(g) + i));
      minw = min(minw, w);
      if (w > maxw) {
        maxw = w;
        imax = i;
      }
    }
    const int wmin = __reduce_min_sync(0xffffffffu, minw);
    const int wmax = __reduce_max_sync(0xffffffffu, maxw);
    const uint32_t bal = __ballot_sync(0xffffffffu, maxw == wmax);
    const uint32_t wimax = __shfl_sync(0xffffffffu, imax, __ffs(bal) - 1);
    if (lane == 0) {
      s_min[warp] = wmin;
      s_max[warp] = wmax;
      s_imax[warp] = wimax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int mn = s_min[0], mx = s_max[0];
      uint32_t im = s_imax[0];
      for (int k = 1; k < kWarps; ++k) {
        mn = min(mn, s_min[k]);
        if (s_max[k] > mx) {
          mx = s_max[k];
          im = s_imax[k];
        }
      }
      V val;
      round1_finish<V>(p, u, p0, mn, mx, im, val);
      ++L.visits;
      ++L.apps;
      L.edges += e - b;
      if (val > V(0)) {
        set_bit(p, chg, u);
        if (p.r1_cand) set_bit(p, p.cand, u);
        ++L.phase_count;
        ++L.lifts;
      }
    }
  }
  __syncthreads();
  // medium: one warp per row
  const uint32_t nM = class_size(g, 1);
  WarpClaim wc;
  uint32_t it;
  while (warp_claim(slot_dyn + 0, nM, wc, it)) {
    const uint32_t u = class_item(g, 1, it);
    if (!owned(p, u)) continue;
    const bool p0 = u < g.rb[kP1L];
    const uint32_t b = __ldg(g.off + u), e = __ldg(g.off + u + 1);
    // per-lane min / max / argmax over a 128-edge stride (4 independent
    // loads in flight), one warp reduction at the end
    int lmin = INT32_MAX, lmax = INT32_MIN;
    uint32_t limax = b;
    for (uint32_t i0 = b; i0 < e; i0 += 128) {
      int wv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t i = i0 + k * 32 + lane;
        wv[k] = i < e ? rec_w(g, __ldcs(erecs(g) + i)) : INT32_MIN;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t i = i0 + k * 32 + lane;
        if (i < e) {
          lmin = min(lmin, wv[k]);
          if (wv[k] > lmax) {
            lmax = wv[k];
            limax = i;
          }
        }
      }
      if (p0 && __any_sync(0xffffffffu, lmax >= 0)) break;  // a satisfied move
    }
    const int minw = __reduce_min_sync(0xffffffffu, lmin);
    const int maxw = __reduce_max_sync(0xffffffffu, lmax);
    const uint32_t imax = __shfl_sync(0xffffffffu, limax,
                                      __ffs(__ballot_sync(0xffffffffu, lmax == maxw)) - 1);
    if (lane == 0) {
      V val;
      round1_finish<V>(p, u, p0, minw, maxw, imax, val);
      ++L.visits;
      ++L.apps;
      L.edges += e - b;
      if (val > V(0)) {
        set_bit(p, chg, u);
        if (p.r1_cand) set_bit(p, p.cand, u);
        ++L.phase_count;
        ++L.lifts;
      }
    }
  }
  block_flush(L, sum_dst);
}

// Player-1 light rows: sorted by weight at upload (egs_build.cuh
// k_sort_p1_rows), so delta(0)(v) = max(0, -w_min) is the first record's,
// which the upload mirrors into g.rec0[v] -- no row is streamed: 4 (8) bytes
// per vertex, coalesced, where a row read costs a 32-byte sector.  A warp
// takes kR1Words bitmap words (32 vertices each) per step and issues all
// their loads before using any.
constexpr int kR1Words = 4;
#ifndef EGS_R1_PAIRS
#define EGS_R1_PAIRS 1
#endif
constexpr bool kR1Pairs = EGS_R1_PAIRS != 0;  // round1_p0_pairs
template <class V>
__device__ __noinline__ void round1_p1_light(const SolveParams<V>& p, uint32_t lo, uint32_t hi,
                                             uint32_t* chg, unsigned int* sum_dst) {
  const Graph& g = p.g;
  Local L;
  if (hi > lo) {
    const uint32_t nwarps = gridDim.x * kWarps;
    const uint32_t gw = (blockIdx.x * kBlock + threadIdx.x) >> 5, lane = lane_id();
    const uint32_t w_lo = lo >> 5, w_hi = (hi + 31) >> 5;
    for (uint32_t w0 = w_lo + gw * kR1Words; w0 < w_hi; w0 += nwarps * kR1Words) {
      bool in[kR1Words];
      ERec r[kR1Words];
      uint32_t eb = 0, ee = 0;  // lane k < kR1Words: the edge span of word w0 + k's rows
#pragma unroll
      for (int k = 0; k < kR1Words; ++k) {
        const uint32_t v = ((w0 + k) << 5) + lane;
        in[k] = w0 + k < w_hi && v >= lo && v < hi;
        r[k] = in[k] ? __ldcs(static_cast<const ERec*>(g.rec0) + v) : ERec{};
      }
      if (lane < (uint32_t)kR1Words && w0 + lane < w_hi) {
        eb = __ldg(g.off + max(lo, (w0 + lane) << 5));
        ee = __ldg(g.off + min(hi, ((w0 + lane) << 5) + 32));
      }
      L.edges += ee - eb;  // one lift application relaxes the row
#pragma unroll
      for (int k = 0; k < kR1Words; ++k) {
        const uint32_t v = ((w0 + k) << 5) + lane;
        bool ch = false;
        if (in[k]) {
          const V val = ominus_cap<V>(V(0), rec_w(g, r[k]), g.cap);
          ++L.visits;
          ++L.apps;
          if (val > V(0)) {
            r1_store<V>(p, v, val);
            ++L.lifts;
            ch = true;
          }
        }
        const uint32_t m = __ballot_sync(0xffffffffu, ch);
        if (m && lane == 0 && w0 + k < w_hi) bits_or(p, chg + w0 + k, m);
        if (w0 + k < w_hi) r1_cand_bits<V>(p, w0 + k, m);
        L.phase_count += ch;
      }
    }
  }
  block_flush(L, sum_dst);
}

template <class V>
__device__ __noinline__ void phase_round1(const SolveParams<V>& p, uint32_t* chg,
                                          unsigned int* slot_sum, unsigned int* slot_dyn) {
  const Graph& g = p.g;
  round1_long<V>(p, chg, slot_sum + 0, slot_dyn);
  // player-0 light rows stream through the tile pipeline (their witness
  // needs the whole row); player-1 light rows read their first record
  if (kR1Pairs && kStages == 2 && kPackedWitnessKey && g.tbits >= 5 &&
      (p.use_tma & kTmaRound1) != 0)
    round1_p0_pairs<V>(p, clip_lo(p, g.rb[kP0L]), clip_hi(p, g.rb[kP0M]),
                       slot_dyn + kTileCursor, chg, slot_sum + 0);
  else
    round1_light<V>(p, clip_lo(p, g.rb[kP0L]), clip_hi(p, g.rb[kP0M]), 0u, 0u,
                    slot_dyn + kTileCursor, chg, slot_sum + 0);
  round1_p1_light<V>(p, clip_lo(p, g.rb[kP1L]), clip_hi(p, g.rb[kP1M]), chg, slot_sum + 0);
}

// One lift round.  Dense (Jacobi): every vertex, raised values staged for
// the commit phase.  Sparse (solve_frontier, solver_par.cpp:389-417): the
// vertices of frontier `cur`, lifted in place, each raised vertex pushing its
// predecessors into frontier `nxt` -- one phase per sparse round.  Raised
// vertices are marked in `chg`; the other round's bitmap is cleared for
// reuse.  The produced frontier's size goes to slot_sum[2], its queued long
// columns to slot_dyn[2].
template <class V>
__device__ __noinline__ void phase_lift(const SolveParams<V>& p, bool dense, Frontier cur,
                                        Frontier nxt, unsigned int* cnt_after,
                                        uint32_t* chg, uint32_t* other,
                                        unsigned int* slot_sum, unsigned int* slot_dyn,
                                        bool sweep = false, bool p1_listed = false) {
  const Graph& g = p.g;
  const uint32_t tid = blockIdx.x * kBlock + threadIdx.x;
  const uint32_t nthreads = gridDim.x * kBlock;
  const uint32_t nwords = (g.n + 31) >> 5;
  Local L;
  unsigned int* sum_dst = slot_sum + 0;
  for (uint32_t w = tid; w < nwords; w += nthreads) {
    other[w] = 0u;
    if (dense) {  // no frontier survives a dense round
      p.frb[0][w] = 0u;
      p.frb[1][w] = 0u;
    }
  }
  if (dense) {
    // sweep: every vertex lifted IN PLACE, reading whatever its successors
    // hold at that moment -- the reference's solve_sweep (solver_par.cpp:
    // 205-228, clamped atomic store); otherwise Jacobi (staged, committed)
    SubTimer st(p.ctr, p.trace != nullptr);
    block_rows<V>(p, class_size(g, 2), slot_dyn + 1,
                  [gp = &g](uint32_t i) { return class_item(*gp, 2, i); }, chg, sum_dst, false,
                  Frontier{}, nullptr, nullptr, sweep);
    st.lap(kSubHeavy);
    warp_rows<V>(p, class_size(g, 1), slot_dyn + 0,
                 [gp = &g](uint32_t i) { return class_item(*gp, 1, i); }, chg, sum_dst, false,
                 Frontier{}, nullptr, nullptr, sweep);
    st.lap(kSubMedium);
    if (sweep) {
      dense_light_p0<V, true>(p, clip_lo(p, g.rb[kP0L]), clip_hi(p, g.rb[kP0M]), chg, sum_dst);
      st.lap(kSubLightP0);
      dense_light_p1<V, true>(p, clip_lo(p, g.rb[kP1L]), clip_hi(p, g.rb[kP1M]),
                              slot_dyn + kTileCursor, chg, sum_dst);
    } else {
      dense_light_p0<V>(p, clip_lo(p, g.rb[kP0L]), clip_hi(p, g.rb[kP0M]), chg, sum_dst);
      st.lap(kSubLightP0);
      if (p1_listed)
        dense_light_p1_listed<V>(p, p.fr[0], vload(&p.sh->p1live), chg, sum_dst);
      else
        dense_light_p1<V>(p, clip_lo(p, g.rb[kP1L]), clip_hi(p, g.rb[kP1M]),
                          slot_dyn + kTileCursor, chg, sum_dst);
    }
    st.lap(kSubLightP1);
  } else {
    if (blockIdx.x == 0 && threadIdx.x < 3) cnt_after[threadIdx.x] = 0u;
    const uint32_t cL = vload(cur.cnt + 0);
    const uint32_t cM = vload(cur.cnt + 1);
    const uint32_t cH = vload(cur.cnt + 2);
    const uint32_t* lL = cur.list[0];
    const uint32_t* lM = cur.list[1];
    const uint32_t* lH = cur.list[2];
    unsigned int* act_dst = slot_sum + 2;
    unsigned int* qlong = slot_dyn + 2;
    SubTimer st(p.ctr, p.trace != nullptr);
    block_rows<V>(p, cH, slot_dyn + 1, [=](uint32_t i) { return ldcg(lH + i); }, chg, sum_dst,
                  true, nxt, qlong, act_dst);
    st.lap(kSubHeavy);
    warp_rows<V>(p, cM, slot_dyn + 0, [=](uint32_t i) { return ldcg(lM + i); }, chg, sum_dst,
                 true, nxt, qlong, act_dst);
    st.lap(kSubMedium);
    sparse_light<V>(p, lL, cL, chg, sum_dst, nxt, qlong, act_dst);
    st.lap(kSubSparseLight);
    // leave this frontier's membership bits clear for the token after next
    for (uint32_t i = tid; i < cL + cM + cH; i += nthreads) {
      const uint32_t v = i < cL        ? ldcg(lL + i)
                         : i < cL + cM ? ldcg(lM + (i - cL))
                                       : ldcg(lH + (i - cL - cM));
      atomicAnd(cur.frb + (v >> 5), ~(1u << (v & 31u)));
    }
    if (tid == 0) L.pops += cL + cM + cH;
  }
  block_flush(L, sum_dst);
}

// Commit of a Jacobi round: every vertex raised in the round (marked in
// `chg`) takes its staged value.  Lifts of the round all read the measure
// of the previous round, exactly the synchronous rounds of solve_frontier /
// solve_sweep (solver_par.cpp:205-228, 389-417).
// The staged values of a commit step: only those of raised vertices (their
// chg bit first), or -- when many vertices were raised (`dense`) -- every
// slot at once, independent of the bitmap words so both loads are in flight
// together; the caller reads val[k] only where the bit is set.
template <class V, int U>
__device__ __forceinline__ void commit_stage_loads(const SolveParams<V>& p, bool dense,
                                                   uint32_t w0, uint32_t whi, uint32_t lane,
                                                   const uint32_t (&bits)[U], V (&val)[U],
                                                   V other) {
  if (dense) {
#pragma unroll
    for (int k = 0; k < U; ++k)
      val[k] = ((w0 + k) << 5) + lane < p.g.n ? ldcg(p.stage + ((w0 + k) << 5) + lane) : other;
  } else {
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint32_t v = ((w0 + k) << 5) + lane;
      val[k] = ((bits[k] >> lane) & 1u) ? ldcg(p.stage + v) : other;
    }
  }
}

// debug_checks (the reference's check_monotone, solver_par.cpp:116-124,179):
// a value the next commit publishes must be above the one it replaces.  Run
// as a phase of its own right before the commit (reads only).
template <class V>
__device__ __noinline__ void phase_debug_raise(const SolveParams<V>& p, const uint32_t* chg) {
  const uint32_t nwarps = gridDim.x * kWarps;
  const uint32_t gw = (blockIdx.x * kBlock + threadIdx.x) >> 5, lane = lane_id();
  for (uint32_t w = (p.own_lo >> 5) + gw; w < ((p.own_hi + 31) >> 5); w += nwarps) {
    const uint32_t v = (w << 5) + lane;
    if (((ldcg(chg + w) & own_mask(p, w)) >> lane) & 1u) {
      if (!(ldcg(p.stage + v) > ldcg(p.f + v))) atomicOr(&p.sh->bad, 1u);
    }
  }
}

template <class V, bool MULTI>
__device__ __noinline__ void phase_commit(const SolveParams<V>& p, const uint32_t* chg,
                                          bool dense = false) {
  constexpr int U = 8;  // words per warp step, all loads issued before any store
  const uint32_t n = p.g.n;
  const uint32_t nwords = (n + 31) >> 5;
  const uint32_t nwarps = gridDim.x * kWarps;
  const uint32_t gw = (blockIdx.x * kBlock + threadIdx.x) >> 5;
  const uint32_t lane = lane_id();
  const uint32_t wlo = p.own_lo >> 5, whi = min(nwords, (p.own_hi + 31) >> 5);
  // (scalars of p read once: stores through p.f may alias p for the compiler;
  // one rank or several is a template parameter)
  V* const f = p.f;
  for (uint32_t w0 = wlo + gw * U; w0 < whi; w0 += nwarps * U) {
    uint32_t bits[U];
    V val[U];
#pragma unroll
    for (int k = 0; k < U; ++k)
      bits[k] = w0 + k < whi ? ldcg(chg + w0 + k) & (MULTI ? own_mask(p, w0 + k) : ~0u) : 0u;
    commit_stage_loads<V, U>(p, dense, w0, whi, lane, bits, val, V(0));
#pragma unroll
    for (int k = 0; k < U; ++k)
      if ((bits[k] >> lane) & 1u) {
        if (MULTI)
          f_put<V>(p, ((w0 + k) << 5) + lane, val[k]);
        else
          stcg(f + ((w0 + k) << 5) + lane, val[k]);
      }
  }
}

// Certificate, step 1: the candidates are the non-top vertices raised in the
// round just finished (`chg`): losing vertices keep climbing, and starting
// from any subset is sound (the pruned set is still closed).  Candidate
// bits go to p.cand, one word per 32 vertices.
template <class V>
__device__ __noinline__ void phase_cert_init(const SolveParams<V>& p, const uint32_t* chg,
                                             unsigned int* slot_sum) {
  const uint32_t tid = blockIdx.x * kBlock + threadIdx.x;
  const uint32_t nthreads = gridDim.x * kBlock;
  const uint32_t nwarps = gridDim.x * kWarps;
  const uint32_t gw = tid >> 5, lane = lane_id();
  Local L;
  for (uint32_t w = tid; w < ((p.g.n + 31) >> 5); w += nthreads) p.rbm[1][w] = 0u;
  const uint32_t wlo = p.own_lo >> 5, whi = (p.own_hi + 31) >> 5;
  for (uint32_t w = wlo + gw; w < whi; w += nwarps) {
    const uint32_t v = (w << 5) + lane;
    const uint32_t bits = ldcg(chg + w);
    const bool in = v >= p.own_lo && v < p.own_hi;
    const V fv = in ? ldcg(p.f + v) : Top<V>::v;
    const bool c = in && ((bits >> lane) & 1u) && fv != Top<V>::v;
    if (c) f_put<V>(p, v, fv | CandFlag<V>::v);
    const uint32_t m = __ballot_sync(0xffffffffu, c);
    if (lane == 0) stcg(p.cand + w, m);
  }
  block_flush(L, slot_sum + 1);
}

// Commit fused with certificate step 1 (one pass over the words of `chg`
// instead of two): a raised vertex publishes its staged value and, unless it
// reached top, becomes a candidate (bit + mark).
template <class V, bool MULTI>
__device__ __noinline__ void phase_commit_cert_init(const SolveParams<V>& p, const uint32_t* chg,
                                                    bool dense = false) {
  constexpr V TOP = Top<V>::v;
  constexpr int U = 8;  // words per warp step, all loads issued before any store
  const uint32_t nwords = (p.g.n + 31) >> 5;
  const uint32_t nwarps = gridDim.x * kWarps;
  const uint32_t tid = blockIdx.x * kBlock + threadIdx.x;
  const uint32_t gw = tid >> 5, lane = lane_id();
  for (uint32_t w = tid; w < nwords; w += gridDim.x * kBlock) p.rbm[1][w] = 0u;
  const uint32_t wlo = p.own_lo >> 5, whi = min(nwords, (p.own_hi + 31) >> 5);
  V* const f = p.f;
  uint32_t* const cand = p.cand;
  for (uint32_t w0 = wlo + gw * U; w0 < whi; w0 += nwarps * U) {
    uint32_t bits[U];
    V val[U];
#pragma unroll
    for (int k = 0; k < U; ++k)
      bits[k] = w0 + k < whi ? ldcg(chg + w0 + k) & (MULTI ? own_mask(p, w0 + k) : ~0u) : 0u;
    commit_stage_loads<V, U>(p, dense, w0, whi, lane, bits, val, TOP);
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (w0 + k >= whi) break;
      const bool raised = (bits[k] >> lane) & 1u;
      const bool c = raised && val[k] != TOP;
      const V x = c ? val[k] | CandFlag<V>::v : val[k];
      if (raised) {
        if (MULTI)
          f_put<V>(p, ((w0 + k) << 5) + lane, x);
        else
          stcg(f + ((w0 + k) << 5) + lane, x);
      }
      const uint32_t m = __ballot_sync(0xffffffffu, c);
      if (lane == 0) stcg(cand + w0 + k, m);
    }
  }
}

// Certificate, step 2: pruning passes.  A removed candidate loses its bit
// in p.cand and its mark in f and gets a bit in `rbm` (removed in this pass), so the next pass
// can be sparse: only candidate predecessors of this pass's removals
// (phase_cert_mark, via the CSC) can lose their condition.

// One candidate, evaluated by the lanes a row's class gets; returns removed.
template <class V>
__device__ __forceinline__ bool cert_check_thread(const SolveParams<V>& p, uint32_t v, Local& L) {
  if (!cand_bit(p, v)) return false;
  const int64_t fv = cand_value<V>(ldcg(p.f + v));
  const bool keep = v < p.g.rb[kP1L] ? cert_keep_thread<V, true>(p, v, fv, L)
                                     : cert_keep_thread<V, false>(p, v, fv, L);
  ++L.cert_scanned;
  if (!keep) cand_clear(p, v, fv);
  return !keep;
}

// Heavy (CTA) and medium (warp) candidates from an item source; removal
// bits go to `rbm`.  Block-uniform.
template <class V, class ItemsH, class ItemsM>
__device__ __forceinline__ void cert_long_rows(const SolveParams<V>& p, uint32_t nH,
                                               ItemsH itemsH, uint32_t nM, ItemsM itemsM,
                                               unsigned int* slot_dyn, uint32_t* rbm, Local& L,
                                               WarpLists& q, const Frontier& qt) {
  __shared__ unsigned int s_item;
  const Graph& g = p.g;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_item = atomicAdd(slot_dyn + 1, 1u);
    __syncthreads();
    const uint32_t i = s_item;
    if (i >= nH) break;
    const uint32_t v = itemsH(i);
    if (!owned(p, v)) continue;
    if (!cand_bit(p, v)) continue;
    const int64_t fv = cand_value<V>(ldcg(p.f + v));
    const bool keep = v < g.rb[kP1L] ? cert_keep_block<V, true>(p, v, fv, L)
                                     : cert_keep_block<V, false>(p, v, fv, L);
    if (threadIdx.x == 0) {
      ++L.cert_scanned;
      if (!keep) {
        cand_clear(p, v, fv);
        set_bit(p, rbm, v);
        ++L.phase_count;
      }
    }
    if (threadIdx.x < 32) push_cert_preds<V>(p, !keep && threadIdx.x == 0, v, q, qt, L);
  }
  __syncthreads();
  WarpClaim wc;
  uint32_t i;
  while (warp_claim(slot_dyn + 0, nM, wc, i)) {
    const uint32_t v = itemsM(i);
    if (!owned(p, v)) continue;
    if (!cand_bit(p, v)) continue;
    const int64_t fv = cand_value<V>(ldcg(p.f + v));
    const bool keep = v < g.rb[kP1L] ? cert_keep_warp<V, true>(p, v, fv, L)
                                     : cert_keep_warp<V, false>(p, v, fv, L);
    if (lane_id() == 0) {
      ++L.cert_scanned;
      if (!keep) {
        cand_clear(p, v, fv);
        set_bit(p, rbm, v);
        ++L.phase_count;
      }
    }
    push_cert_preds<V>(p, !keep && lane_id() == 0, v, q, qt, L);
  }
}

// Dense pass over every owned candidate (removed count -> slot_sum[1]).
// `rbm_clear` (the bitmap two passes old) is zeroed for reuse.
template <class V>
__device__ __noinline__ void phase_cert_prune(const SolveParams<V>& p, unsigned int* slot_sum,
                                              unsigned int* slot_dyn, uint32_t* rbm,
                                              uint32_t* rbm_clear, Frontier qt = Frontier{},
                                              uint32_t* qclear = nullptr) {
  const Graph& g = p.g;
  const uint32_t tid = blockIdx.x * kBlock + threadIdx.x;
  const uint32_t nthreads = gridDim.x * kBlock;
  const uint32_t nwords = (g.n + 31) >> 5;
  Local L;
  WarpLists q = warp_lists_small();
  // the cascade that may follow starts from an empty queue and one token
  // per warp (phase_cert_cascade)
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.sh->qhead = 0u;
    p.sh->qtail = 0u;
    p.sh->qpend = gridDim.x * kWarps;
    p.sh->p1live = 0u;  // (the apply that ends this attempt lists into it)
  }
  // (a dense pass leaves the last pass's re-check queue unread: its dedup
  // bitmap is cleared whole)
  for (uint32_t w = tid; w < nwords; w += nthreads) {
    rbm_clear[w] = 0u;
    if (qclear) qclear[w] = 0u;
  }
  auto itH = [gp = &g](uint32_t i) { return class_item(*gp, 2, i); };
  auto itM = [gp = &g](uint32_t i) { return class_item(*gp, 1, i); };
  cert_long_rows<V>(p, class_size(g, 2), itH, class_size(g, 1), itM, slot_dyn, rbm, L, q, qt);
  // light candidates: one row per lane through the TMA tile pipeline (tiles
  // without a candidate are skipped); removals are published in rbm
  {
    auto load = [&](uint32_t v, V& fv) { fv = ldcg(p.f + v); };
    auto test = [&](uint32_t, V) { return true; };  // the tile mask is the candidate word
    // a pass keeps most player-0 candidates, and keeping one reads its whole
    // row: player-0 rows test kCertChunkP0 edges per step, player-1 rows
    // (kept by their first good edge) kCertChunk
    auto scan = [&](auto chunk, bool p0, const ERec* rec, uint32_t len, uint32_t rot,
                    int64_t fv) {
      constexpr int C = decltype(chunk)::value;
      for (uint32_t k0 = 0; k0 < len; k0 += C) {
        int2 r[C];
#pragma unroll
        for (int k = 0; k < C; ++k) {
          uint32_t j = min(k0 + k, len - 1) + rot;
          j = j >= len ? j - len : j;
          r[k] = dec(g, rec[j]);
        }
        V c[C];
#pragma unroll
        for (int k = 0; k < C; ++k) c[k] = gather(p.f + r[k].x);
        bool all = true, any = false;
#pragma unroll
        for (int k = 0; k < C; ++k) {
          const bool gd = good_target<V>(fv, c[k], r[k].y);
          all &= gd;
          any |= gd;
        }
        L.cert_edges += min((uint32_t)C, len - k0);
        if (p0 && !all) return false;
        if (!p0 && any) return true;
      }
      return p0;
    };
    auto row = [&](uint32_t v, const ERec* rec, uint32_t len, uint32_t, V cv) {
      const int64_t fv = cand_value<V>(cv);
      const bool p0 = v < g.rb[kP1L];
      // player-1 rows are sorted by weight (upload): read in order, the most
      // negative -- likeliest good -- edges first (the bank conflicts of
      // unrotated reads cost a few cycles per step; the gathers, microseconds)
      const uint32_t rot = p0 ? row_rot(len) : 0u;
      ++L.cert_scanned;
      const bool keep = p0 ? scan(std::integral_constant<int, kCertChunkP0>{}, true, rec, len,
                                  rot, fv)
                           : scan(std::integral_constant<int, kCertChunk>{}, false, rec, len,
                                  rot, fv);
      if (!keep) cand_clear(p, v, fv);
      return !keep;
    };
    auto fallback = [&](uint32_t v, V) { return cert_check_thread<V>(p, v, L); };
    auto after = [&](uint32_t v, bool removed) { push_cert_preds<V>(p, removed, v, q, qt, L); };
    tma_tiles<V>(p, (p.use_tma & kTmaCert) != 0, clip_lo(p, g.rb[kP0L]), clip_hi(p, g.rb[kP0M]),
                 clip_lo(p, g.rb[kP1L]), clip_hi(p, g.rb[kP1M]), slot_dyn + kTileCursor, p.cand,
                 rbm, L, load, test, row, fallback, after);
  }
  if (qt.cnt)
    for (int c = 0; c < 3; ++c) lists_flush(q, c, qt.list[c], qt.cnt + c);
  block_flush(L, slot_sum + 1);
}

// After a dense pass (which does not push: its removals are many, and the
// pushes would stall its tile pipeline) the first sparse pass's queue is
// built here from the removal bits `rbm_in`: the owned candidate
// predecessors of every removed vertex, once each (dedup t.frb).
template <class V>
__device__ __noinline__ void phase_cert_mark(const SolveParams<V>& p, const uint32_t* rbm_in,
                                             Frontier t, unsigned int* slot_sum) {
  const uint32_t nwords = (p.g.n + 31) >> 5;
  const uint32_t nwarps = gridDim.x * kWarps;
  const uint32_t gw = (blockIdx.x * kBlock + threadIdx.x) >> 5;
  Local L;
  WarpLists q = warp_lists();
  for (uint32_t w0 = gw * 32; w0 < nwords; w0 += nwarps * 32) {
    const uint32_t wi = w0 + lane_id();
    uint32_t bits = wi < nwords ? ldcg(rbm_in + wi) : 0u;
    while (__any_sync(0xffffffffu, bits != 0u)) {
      uint32_t u = 0;
      bool any = false;
      if (bits) {
        u = (wi << 5) + (__ffs(bits) - 1);
        bits &= bits - 1;
        any = true;
      }
      push_cert_preds<V>(p, any, u, q, t, L);
    }
  }
  for (int c = 0; c < 3; ++c) lists_flush(q, c, t.list[c], t.cnt + c);
  block_flush(L, slot_sum + 2);
}

// Sparse pass: re-check the queued candidates -- the candidate predecessors
// of the last pass's removals, pushed by that pass (queue `cur`, counts
// qcnt) -- and push the candidate predecessors of this pass's removals into
// queue `nxt`; removed -> slot_sum[1], bits -> rbm.  Clears the dedup bits of
// the entries it reads and the stale bitmap rbm_clear.
template <class V>
__device__ __noinline__ void phase_cert_check(const SolveParams<V>& p, Frontier cur,
                                              const unsigned int* qcnt, unsigned int* slot_sum,
                                              unsigned int* slot_dyn, uint32_t* rbm,
                                              uint32_t* rbm_clear, Frontier nxt) {
  const uint32_t tid = blockIdx.x * kBlock + threadIdx.x;
  const uint32_t nthreads = gridDim.x * kBlock;
  const uint32_t nwords = (p.g.n + 31) >> 5;
  Local L;
  WarpLists q = warp_lists_small();
  for (uint32_t w = tid; w < nwords; w += nthreads) rbm_clear[w] = 0u;
  const uint32_t cL = vload(qcnt + 0);
  const uint32_t cM = vload(qcnt + 1);
  const uint32_t cH = vload(qcnt + 2);
  const uint32_t* lL = cur.list[0];
  const uint32_t* lM = cur.list[1];
  const uint32_t* lH = cur.list[2];
  auto itH = [=](uint32_t i) { return ldcg(lH + i); };
  auto itM = [=](uint32_t i) { return ldcg(lM + i); };
  // several ranks: no pushes (the next pass is built by phase_cert_mark)
  if (p.world > 1) nxt = Frontier{};
  cert_long_rows<V>(p, cH, itH, cM, itM, slot_dyn, rbm, L, q, nxt);
  for (uint32_t i0 = blockIdx.x * kBlock + (threadIdx.x & ~31u); i0 < cL; i0 += nthreads) {
    const uint32_t i = i0 + lane_id();
    uint32_t v = 0;
    bool removed = false;
    if (i < cL) {
      v = ldcg(lL + i);
      removed = cert_check_thread<V>(p, v, L);
    }
    if (removed) {
      set_bit(p, rbm, v);
      ++L.phase_count;
    }
    push_cert_preds<V>(p, removed, v, q, nxt, L);
  }
  if (nxt.cnt)
    for (int c = 0; c < 3; ++c) lists_flush(q, c, nxt.list[c], nxt.cnt + c);
  for (uint32_t i = tid; i < cL + cM + cH; i += nthreads) {
    const uint32_t v = i < cL ? ldcg(lL + i) : i < cL + cM ? ldcg(lM + (i - cL)) : ldcg(lH + (i - cL - cM));
    atomicAnd(cur.frb + (v >> 5), ~(1u << (v & 31u)));
  }
  block_flush(L, slot_sum + 1);
}

// Certificate, step 2 (one rank): the cascade after a dense pass, in ONE
// phase instead of a mark phase plus one sparse pass per removal wave.  The
// candidate predecessors of the dense pass's removals (bitmap rbm_in, CSC)
// enter a work queue; warps re-check queued candidates and push the
// candidate predecessors of every removal, until the queue is empty and no
// item is in flight -- the greatest fixpoint of the pruning, reached in any
// order.  The queue is a ring of n slots (p.ring, kRingEmpty when free):
// a producer reserves slots (Scratch::qtail, after counting the items in
// Scratch::qpend) and writes them; a consumer claims a range (qhead, by CAS
// up to qtail), waits for each slot's write, frees it, and only then clears
// the item's dedup bit (qbits) -- so at most one queued copy per vertex and
// at most n unfreed slots, and a vertex whose successor is removed after its
// re-check is queued again.  qpend counts reserved items not yet finished
// (their pushes included) plus one token per warp until its mark step is
// done; every warp leaves when it is zero.  All CTAs are co-resident
// (persistent cooperative launch), so every spin ends.
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <class V>
__device__ __forceinline__ void ring_push(const SolveParams<V>& p, bool add, uint32_t u,
                                          uint32_t n) {
  const uint32_t m = __ballot_sync(0xffffffffu, add);
  if (!m) return;
  uint32_t base = 0;
  if (lane_id() == 0) {
    atomicAdd(&p.sh->qpend, (unsigned int)__popc(m));
    base = atomicAdd(&p.sh->qtail, (unsigned int)__popc(m));
  }
  base = __shfl_sync(0xffffffffu, base, 0);
  if (add) {
    const uint32_t slot = (base + __popc(m & lanemask_lt())) % p.ring_cap;
    // the slot's previous item (one lap back) is claimed already (at most n
    // items are queued, each holding its dedup bit); wait until its consumer
    // frees it.  A warp pushes only after freeing its own claims, and a
    // consumer waits only for an earlier reservation's write: no cycle.
    while (ld_relaxed_gpu(p.ring + slot) != kRingEmpty) __nanosleep(32);
    __stcg(p.ring + slot, u);
  }
}

// the candidate predecessors of the lanes with `removed` (their CSC columns,
// expanded by the warp), each queued once (dedup bits qbits).  Warp-uniform.
template <class V>
__device__ __forceinline__ void cascade_push_preds(const SolveParams<V>& p, bool removed,
                                                   uint32_t v, uint32_t* qbits) {
  if (!__any_sync(0xffffffffu, removed)) return;
  // the removal (bit and mark cleared) is visible before any queue bit is
  // touched: a predecessor still queued (its bit found set) is re-checked
  // after its consumer clears that bit, and then sees the removal
  __threadfence();
  uint32_t b = 0, e = 0;
  if (removed) {
    b = __ldg(p.g.coff + v);
    e = __ldg(p.g.coff + v + 1);
  }
  warp_expand(b, e, [&](bool valid, uint32_t idx, uint32_t) {
    bool add = false;
    uint32_t u = 0;
    if (valid) {
      u = __ldg(p.g.csrc + idx);
      const uint32_t bit = 1u << (u & 31u);
      add = ((ldcg(p.cand + (u >> 5)) & bit) != 0) && !(ldcg(qbits + (u >> 5)) & bit) &&
            !(atomicOr(qbits + (u >> 5), bit) & bit);
    }
    ring_push<V>(p, add, u, p.g.n);
  });
}

template <class V>
__device__ __noinline__ void phase_cert_cascade(const SolveParams<V>& p, const uint32_t* rbm_in,
                                                uint32_t* qbits, unsigned int* slot_sum) {
  const uint32_t n = p.g.n;
  const uint32_t nwords = (n + 31) >> 5;
  const uint32_t nwarps = gridDim.x * kWarps;
  const uint32_t gw = (blockIdx.x * kBlock + threadIdx.x) >> 5, lane = lane_id();
  Scratch* sh = p.sh;
  Local L;
  // mark: the candidate predecessors of the dense pass's removals
  for (uint32_t w0 = gw * 32; w0 < nwords; w0 += nwarps * 32) {
    const uint32_t wi = w0 + lane;
    uint32_t bits = wi < nwords ? ldcg(rbm_in + wi) : 0u;
    while (__any_sync(0xffffffffu, bits != 0u)) {
      uint32_t u = 0;
      bool any = false;
      if (bits) {
        u = (wi << 5) + (__ffs(bits) - 1);
        bits &= bits - 1;
        any = true;
      }
      cascade_push_preds<V>(p, any, u, qbits);
    }
  }
  if (lane == 0) atomicSub(&sh->qpend, 1u);  // this warp's mark token
  // drain: every lane holds one queue position at a time (claimed with one
  // atomicAdd per warp for the lanes that need one, possibly past the
  // reserved positions) and polls it; lanes whose item has arrived re-check
  // it, push, and take a new position.  A lane never blocks on its
  // position, so an item is never waited for by the warp that must finish
  // it.  When no item is in flight every held position is past the last
  // reserved one (a reserved position's item is unfinished until its holder
  // processes it), and the warp leaves.
  const uint32_t cap = p.ring_cap;
  constexpr uint32_t kNoPos = 0xFFFFFFFFu;
  uint32_t pos = kNoPos;
  unsigned ns = 32;
  for (;;) {
    const uint32_t need = __ballot_sync(0xffffffffu, pos == kNoPos);
    if (need) {
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&sh->qhead, (unsigned int)__popc(need));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (pos == kNoPos) pos = base + __popc(need & lanemask_lt());
    }
    uint32_t* s = p.ring + pos % cap;
    uint32_t v = ld_relaxed_gpu(s);
    const bool have = v != kRingEmpty;
    if (have) {
      __stcg(s, kRingEmpty);
      __threadfence();
      atomicAnd(qbits + (v >> 5), ~(1u << (v & 31u)));
      __threadfence();  // (pairs with the pusher's fence: see its removal)
      pos = kNoPos;
    }
    const uint32_t got = __ballot_sync(0xffffffffu, have);
    if (!got) {
      if (ld_relaxed_gpu(&sh->qpend) == 0u) break;  // nothing in flight: done
      __nanosleep(ns);
      ns = ns < 1024 ? ns * 2 : 1024;
      continue;
    }
    ns = 32;
    const uint32_t k = __popc(got);
    // light candidates one per lane; medium / heavy ones by the whole warp
    const bool light = have && size_class(p.g, v) == 0;
    bool removed = false;
    if (light) removed = cert_check_thread<V>(p, v, L);
    uint32_t longm = __ballot_sync(0xffffffffu, have && !light);
    while (longm) {
      const int src = __ffs(longm) - 1;
      longm &= longm - 1;
      const uint32_t u = __shfl_sync(0xffffffffu, v, src);
      if (!cand_bit(p, u)) continue;  // warp-uniform
      const int64_t fu = cand_value<V>(ldcg(p.f + u));
      const bool keep = u < p.g.rb[kP1L] ? cert_keep_warp<V, true>(p, u, fu, L)
                                         : cert_keep_warp<V, false>(p, u, fu, L);
      if (lane == src) {
        ++L.cert_scanned;
        if (!keep) cand_clear(p, u, fu);
        removed = !keep;
      }
    }
    L.phase_count += removed;
    cascade_push_preds<V>(p, removed, v, qbits);
    __syncwarp();
    if (lane == 0) atomicSub(&sh->qpend, k);
  }
  block_flush(L, slot_sum + 1);
}

// Certificate, step 3: certified vertices jump to top and count as changed
// in this round so their predecessors are re-lifted (count -> slot_sum[0]).
template <class V, bool MULTI>
__device__ __noinline__ void phase_cert_apply(const SolveParams<V>& p, uint32_t* chg,
                                              unsigned int* slot_sum) {
  const uint32_t nwarps = gridDim.x * kWarps;
  const uint32_t gw = (blockIdx.x * kBlock + threadIdx.x) >> 5;
  const uint32_t lane = lane_id();
  Local L;
  constexpr uint32_t U = 8;  // words per warp step, loads issued together
  const uint32_t w_lo = p.own_lo >> 5, w_hi = (p.own_hi + 31) >> 5;
  V* const f = p.f;
  // the player-1 light vertices left below top are listed for the next
  // (dense) round, which then lifts only them among player-1 light rows
  const uint32_t l1_lo = max(p.g.rb[kP1L], p.own_lo), l1_hi = min(p.g.rb[kP1M], p.own_hi);
  for (uint32_t w0 = w_lo + gw * U; w0 < w_hi; w0 += nwarps * U) {
    uint32_t m[U];
#pragma unroll
    for (uint32_t k = 0; k < U; ++k) m[k] = w0 + k < w_hi ? ldcg(p.cand + w0 + k) : 0u;
    if (((w0 + U) << 5) > l1_lo && (w0 << 5) < l1_hi) {  // warp-uniform
      V fv[U];
#pragma unroll
      for (uint32_t k = 0; k < U; ++k) {
        const uint32_t v = ((w0 + k) << 5) + lane;
        fv[k] = v >= l1_lo && v < l1_hi ? ldcg(f + v) : Top<V>::v;
      }
      uint32_t b[U], tot = 0;
#pragma unroll
      for (uint32_t k = 0; k < U; ++k) {
        b[k] = __ballot_sync(0xffffffffu, fv[k] != Top<V>::v && !((m[k] >> lane) & 1u));
        tot += __popc(b[k]);
      }
      if (tot) {  // one reservation per warp step
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&p.sh->p1live, tot);
        base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
        for (uint32_t k = 0; k < U; ++k) {
          if ((b[k] >> lane) & 1u)
            p.fr[0][base + __popc(b[k] & lanemask_lt())] = ((w0 + k) << 5) + lane;
          base += __popc(b[k]);
        }
      }
    }
#pragma unroll
    for (uint32_t k = 0; k < U; ++k) {
      const bool hit = (m[k] >> lane) & 1u;  // candidate words hold owned, non-top ids only
      if (MULTI) {
        if (hit) f_put<V>(p, ((w0 + k) << 5) + lane, Top<V>::v);
        if (m[k] && lane == 0) bits_or(p, chg + w0 + k, m[k]);
      } else {
        if (hit) stcg(f + ((w0 + k) << 5) + lane, Top<V>::v);
        if (m[k] && lane == 0) atomicOr(chg + w0 + k, m[k]);
      }
      L.phase_count += hit;
      L.certified += hit;
    }
  }
  block_flush(L, slot_sum + 0);
}

template <class V>
__device__ __noinline__ void phase_activate(const SolveParams<V>& p, const uint32_t* chg,
                                            Frontier t, uint32_t* frb_other,
                                            unsigned int* cnt_next, unsigned int* slot_sum,
                                            unsigned int* qlong) {
  const Graph& g = p.g;
  const uint32_t nwords = (g.n + 31) >> 5;
  const uint32_t nwarps = gridDim.x * kWarps;
  const uint32_t gw = (blockIdx.x * kBlock + threadIdx.x) >> 5;
  Local L;
  WarpLists q = warp_lists();
  // the other frontier bitmap may hold a discarded frontier's marks; the
  // counters of the token after this one start at zero
  for (uint32_t w = blockIdx.x * kBlock + threadIdx.x; w < nwords; w += gridDim.x * kBlock)
    frb_other[w] = 0u;
  if (blockIdx.x == 0 && threadIdx.x < 3) cnt_next[threadIdx.x] = 0u;
  for (uint32_t w0 = gw * 32; w0 < nwords; w0 += nwarps * 32) {
    const uint32_t wi = w0 + lane_id();
    uint32_t bits = wi < nwords ? ldcg(chg + wi) : 0u;
    while (__any_sync(0xffffffffu, bits != 0u)) {
      uint32_t b = 0, e = 0;
      if (bits) {
        const uint32_t v = (wi << 5) + (__ffs(bits) - 1);
        bits &= bits - 1;
        b = __ldg(g.coff + v);
        e = __ldg(g.coff + v + 1);
        if (e - b > kLongCol) {
          const uint32_t k = atomicAdd(qlong, 1u);
          p.longcol[2 * k] = v;
          p.longcol[2 * k + 1] = 0u;  // this column's chunk cursor
          e = b;
        }
      }
      expand_preds<V>(p, b, e, q, t, L, false, false);
    }
  }
  for (int c = 0; c < 3; ++c) lists_flush(q, c, t.list[c], t.cnt + c);
  block_flush(L, slot_sum + 2);
}

// The long columns queued by phase_activate: every warp walks the queue and
// claims kColChunk-entry chunks of each column from its cursor.
template <class V>
__device__ __noinline__ void phase_activate_long(const SolveParams<V>& p, Frontier t,
                                                 uint32_t ncols, unsigned int* slot_sum) {
  const Graph& g = p.g;
  Local L;
  WarpLists q = warp_lists();
  for (uint32_t k = 0; k < ncols; ++k) {
    const uint32_t v = ldcg(p.longcol + 2 * k);
    const uint32_t b = __ldg(g.coff + v), e = __ldg(g.coff + v + 1);
    const uint32_t nch = (e - b + kColChunk - 1) / kColChunk;
    for (;;) {
      uint32_t c = 0;
      if (lane_id() == 0) c = atomicAdd(p.longcol + 2 * k + 1, 1u);
      c = __shfl_sync(0xffffffffu, c, 0);
      if (c >= nch) break;
      const uint32_t cb = b + c * kColChunk;
      const uint32_t ce = cb + kColChunk < e ? cb + kColChunk : e;
      for (uint32_t i0 = cb; i0 < ce; i0 += 32)
        activate_pred<V>(p, i0 + lane_id() < ce, i0 + lane_id(), q, t, L);
    }
  }
  for (int c = 0; c < 3; ++c) lists_flush(q, c, t.list[c], t.cnt + c);
  block_flush(L, slot_sum + 2);
}

// ================================================ cross-rank barrier ===
// (multi-GPU, leader thread only, after the grid barrier that ends a phase)
// This rank's phase sums (and its timeout flag) go to every rank's sync
// block, then its arrival epoch with release semantics; it waits for every
// rank's arrival (acquire), and replaces its sums by the global ones, so
// every rank takes the same decision.  Every CTA fenced its peer writes
// (__threadfence_system) before the grid barrier, so they are visible to a
// peer that has seen this arrival.  A peer missing for xwait_ns zeroes the
// sums (the solve winds down) and sets Scratch::xerr.
__device__ __forceinline__ void st_release_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int ld_relaxed_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <class V>
__device__ __noinline__ void xbarrier(const SolveParams<V>& p, unsigned int epoch, unsigned int* slot,
                                      Scratch* sh) {
  XSync* me = p.xsync;
  const int par = epoch & 1;
  const unsigned int mine[4] = {slot[0], slot[1], slot[2], slot[3] + sh->stop};
  for (int q = 0; q < p.world; ++q) {
    XSync* xs = peer_of(p, q, me);
    for (int k = 0; k < 4; ++k) xs->sums[par][p.rank][k] = mine[k];
  }
  __threadfence_system();
  for (int q = 0; q < p.world; ++q) st_release_sys(&peer_of(p, q, me)->arrive[p.rank], epoch);
  const unsigned long long t0 = globaltimer();
  bool late = false;
  for (int q = 0; q < p.world && !late; ++q)
    while ((int)(ld_acquire_sys(&me->arrive[q]) - epoch) < 0) {
      if (globaltimer() - t0 > p.xwait_ns) {
        late = true;
        break;
      }
    }
  if (late) {
    sh->xerr = 1;
    sh->stop = 1;
    for (int k = 0; k < 4; ++k) slot[k] = 0;
    return;
  }
  unsigned int g[4] = {0, 0, 0, 0};
  for (int q = 0; q < p.world; ++q)
    for (int k = 0; k < 4; ++k) g[k] += ld_relaxed_sys(&me->sums[par][q][k]);
  for (int k = 0; k < 3; ++k) slot[k] = g[k];
  sh->stop = g[3] > 0 ? 1u : 0u;
}

// ========================================================== the kernel ===
#ifndef EGS_MIN_BLOCKS
#define EGS_MIN_BLOCKS 2  // resident CTAs per SM: 128 registers, no spills in the lift loops
#endif
template <class V>
__global__ void __launch_bounds__(kBlock, EGS_MIN_BLOCKS)
    k_solve(const __grid_constant__ SolveParams<V> p) {
  cg::grid_group grid = cg::this_grid();
  const Graph& g = p.g;
  const uint32_t n = g.n;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  Scratch* sh = p.sh;
  uint32_t phase = 0;
  // phase timing, kept by the leader thread only: seed, lift, cert, activation
  const unsigned long long t_start = leader ? globaltimer() : 0ull;
  unsigned long long t_prev = t_start;

  auto slot_sum = [&]() { return sh->sum[phase & 3]; };
  auto slot_dyn = [&]() { return sh->dyn[phase & 3]; };
  auto prev_sum = [&](int k) { return vload(&sh->sum[(phase - 1) & 3][k]); };
  // zero the per-phase slots two phases ahead (last read two phases ago)
  auto begin_phase = [&]() {
    if (leader)
      for (int k = 0; k < 8; ++k) {
        if (k < 4) sh->sum[(phase + 2) & 3][k] = 0;
        sh->dyn[(phase + 2) & 3][k] = 0;
      }
    set_phase_slot(slot_sum());
  };
  unsigned int epoch = p.epoch0;  // cross-rank barriers (multi-GPU)
  auto end_phase = [&](int kind, int fine = -1) {
    end_phase_flush();
    if (p.world > 1) __threadfence_system();  // this phase's peer writes, before the barrier
    grid.sync();
    ++phase;
    if (p.world > 1) {
      if (leader) xbarrier<V>(p, ++epoch, sh->sum[(phase - 1) & 3], sh);
      grid.sync();
    }
    if (leader) {
      const unsigned long long t = globaltimer();
      p.ctr[kTimeSeed + kind] += t - t_prev;
      if (fine >= 0) p.ctr[kFineCommit + fine] += t - t_prev;
      if (p.trace && phase < kTraceCap)
        p.trace[phase] = ((unsigned long long)(kind * 8 + fine + 1) << 56) | (t - t_prev);
      t_prev = t;
    }
  };

  tma_init_barriers();
  stats_init();
  if (p.world > 1) {
    // several ranks: this rank's replicated state is reset here, before a
    // cross-rank barrier -- a peer writes into it only after that barrier
    const uint32_t tid = blockIdx.x * kBlock + threadIdx.x, nth = gridDim.x * kBlock;
    const uint32_t words = (n + 31) >> 5;
    for (uint32_t v = tid; v < n; v += nth) p.f[v] = V(0);
    for (uint32_t w = tid; w < words; w += nth) {
      p.chg[0][w] = 0u;
      p.chg[1][w] = 0u;
      p.rbm[0][w] = 0u;
      p.rbm[1][w] = 0u;
    }
    __threadfence_system();
    grid.sync();
    if (leader) xbarrier<V>(p, ++epoch, sh->sum[3], sh);
    grid.sync();
  }

  // ---- round 1: seeding + the first lift, from the weights alone
  begin_phase();
  phase_round1<V>(p, p.chg[0], slot_sum(), slot_dyn());
  end_phase(0);
  uint32_t changed = prev_sum(0);
  unsigned long long round = 1, rounds_dense = 1, rounds_sparse = 0, cert_attempts = 0,
                     cert_passes = 0;
  int K = p.cert_interval > 0 ? p.cert_interval : 1;
  unsigned long long next_cert = (unsigned long long)K;
  unsigned int status = 0;
  // Frontier tokens (struct Frontier): `tok` is the last one consumed or
  // discarded; the next sparse lift reads tok + 1.  `inplace`: the last lift
  // was a sparse round that already pushed frontier tok + 1 (`pushed`
  // entries, `pushed_long` queued long columns).
  unsigned int tok = 0;
  bool inplace = false;
  uint32_t pushed = 0, pushed_long = 0;
  auto frontier = [&](unsigned int k) {
    Frontier t;
    const int b = k & 1;
    for (int c = 0; c < 3; ++c) t.list[c] = p.fr[b] + p.cbase[c];
    t.cnt = sh->fr_cnt[k % 3];
    t.frb = p.frb[b];
    return t;
  };

  for (;;) {
    // `changed` vertices were raised by round `round`, marked in chg
    uint32_t* chg = p.chg[(round - 1) & 1];
    if (changed == 0) break;  // a round that raised nothing: least fixpoint
    // (no attempt in a round that stops the solve: the candidate marks in f
    // never outlive an attempt)
    // (round 1 written straight into f with the candidates marked: the
    // attempt runs whatever the stop flag says, or the marks would outlive it)
    const bool r1d = round == 1 && p.r1_direct;
    const bool cert_now = (r1d && p.r1_cand) || (p.certify && round >= next_cert &&
                                                 round < p.round_budget && !vload(&sh->stop));
    // without a certificate attempt the next round's mode is known already:
    // a sparse next round gets its activation in the commit phase (the
    // activation's top filter may see either the old or the committed value
    // of a predecessor; a stale one only adds a harmless frontier entry)
    const bool fuse_act =
        !inplace && !r1d && !cert_now && !p.no_fuse && p.mode != kModeDense && p.mode != kModeSweep &&
        !(p.mode == kModeAuto && (double)changed * p.avg_in_deg * p.sparse_div >= (double)n);
    if (!inplace && !r1d) {  // a Jacobi round: publish its staged values
      if (p.debug) {  // (its own phase: the commit overwrites what it compares)
        begin_phase();
        phase_debug_raise<V>(p, chg);
        end_phase(1, 0);
      }
      begin_phase();
      // (a commit of many raises loads every staged slot with its bitmap word)
      const bool dense_commit = (uint64_t)changed * kDenseCommitDiv >= n;
      if (cert_now) {  // commit + certificate step 1
        if (p.world > 1)
          phase_commit_cert_init<V, true>(p, chg, dense_commit);
        else
          phase_commit_cert_init<V, false>(p, chg, dense_commit);
      } else {
        if (p.world > 1)
          phase_commit<V, true>(p, chg, dense_commit);
        else
          phase_commit<V, false>(p, chg, dense_commit);
        if (fuse_act)
          phase_activate<V>(p, chg, frontier(tok + 1), p.frb[tok & 1], sh->fr_cnt[(tok + 2) % 3],
                            slot_sum(), slot_dyn() + 2);
      }
      end_phase(1, 0);
    } else if (cert_now && !(r1d && p.r1_cand)) {  // f is current: only mark the candidates
      begin_phase();
      phase_cert_init<V>(p, chg, slot_sum());
      end_phase(2, 1);
    }
    if (round >= p.round_budget) {
      status = 5;
      break;
    }
    if (vload(&sh->stop)) {
      status = 2;
      break;
    }

    // ---- certificate
    bool certified_any = false;
    if (cert_now) {
      ++cert_attempts;
      // pass 1 dense; later passes sparse while the removals are few.  Every
      // pass pushes the candidate predecessors of its removals into the next
      // pass's re-check queue `cq + 1` (lists p.fr[(cq + 1) & 1], dedup bitmap
      // p.cbm[(cq + 1) & 1], counters in the pushing phase's dyn slot 3..5).
      int rb = 1;
      unsigned int cq = 0;
      auto queue = [&](unsigned int k, unsigned int* cnt) {
        Frontier t;
        for (int c = 0; c < 3; ++c) t.list[c] = p.fr[k & 1] + p.cbase[c];
        t.cnt = cnt;
        t.frb = p.cbm[k & 1];
        return t;
      };
      begin_phase();
      phase_cert_prune<V>(p, slot_sum(), slot_dyn(), p.rbm[1], p.rbm[0]);
      end_phase(2, 2);
      ++cert_passes;
      bool queued = false;  // did the last pass push a re-check queue (token cq)?
      uint32_t removed = prev_sum(1);
      while (removed > 0) {
        const bool sparse_pass =
            p.mode != kModeDense && p.mode != kModeSweep &&
            (double)removed * p.avg_in_deg * p.cert_sparse_div < (double)n;
        if (sparse_pass && p.world == 1 && p.cascade) {
          // one rank: the rest of the pruning in one phase (a work queue)
          begin_phase();
          phase_cert_cascade<V>(p, p.rbm[rb], p.cbm[0], slot_sum());
          end_phase(2, 3);
          ++cert_passes;
          break;
        }
        if (sparse_pass) {
          if (!queued) {  // after a dense pass: the queue from its removal bits
            begin_phase();
            phase_cert_mark<V>(p, p.rbm[rb], queue(cq + 1, slot_dyn() + 3), slot_sum());
            end_phase(2, 3);
            ++cq;
          }
          unsigned int* qcnt = sh->dyn[(phase - 1) & 3] + 3;  // the queue's counters
          begin_phase();
          phase_cert_check<V>(p, queue(cq, qcnt), qcnt, slot_sum(), slot_dyn(), p.rbm[rb ^ 1],
                              p.rbm[rb], queue(cq + 1, slot_dyn() + 3));
          end_phase(2, 3);
          ++cq;
          // (several ranks: a pass cannot push the candidate predecessors
          // of the OTHER ranks' removals, so every sparse pass is preceded
          // by a mark phase over the replicated removal bits)
          queued = p.world == 1;
        } else {
          begin_phase();
          phase_cert_prune<V>(p, slot_sum(), slot_dyn(), p.rbm[rb ^ 1], p.rbm[rb], Frontier{},
                              queued ? p.cbm[cq & 1] : nullptr);
          end_phase(2, 2);
          queued = false;
        }
        rb ^= 1;
        ++cert_passes;
        removed = prev_sum(1);
      }
      begin_phase();
      if (p.world > 1)
        phase_cert_apply<V, true>(p, chg, slot_sum());
      else
        phase_cert_apply<V, false>(p, chg, slot_sum());
      end_phase(2, 4);
      const uint32_t cert = prev_sum(0);
      certified_any = cert > 0;
      changed += cert;
      // geometric schedule (rounds 1, 9, 73, 137, ... by default): the first
      // attempt catches the regular climbs (the canonical configs certify
      // their losing region at round 1), later ones get rarer so a game
      // without a climbing region pays O(log) attempts
      K = K * p.cert_growth < 64 ? K * p.cert_growth : 64;
      next_cert = round + (unsigned long long)K;
    }

    // ---- next round: dense, or a frontier of the predecessors of changed
    // vertices (solver_par.cpp:402-410)
    const bool dense =
        p.mode == kModeDense || p.mode == kModeSweep ||
        (p.mode == kModeAuto &&
         (certified_any || (double)changed * p.avg_in_deg * p.sparse_div >= (double)n));
    if (!dense) {
      uint32_t frontier_n, ncols;
      if (inplace && !cert_now && p.world == 1) {  // pushed by the sparse lift
        frontier_n = pushed;
        ncols = pushed_long;
      } else if (fuse_act) {  // produced by the commit phase
        frontier_n = prev_sum(2);
        ncols = vload(sh->dyn[(phase - 1) & 3] + 2);
      } else {
        // a certificate attempt after an in-place round used the frontier
        // lists as its queues: the pushed frontier is discarded and rebuilt
        if (inplace) ++tok;
        begin_phase();
        phase_activate<V>(p, chg, frontier(tok + 1), p.frb[tok & 1], sh->fr_cnt[(tok + 2) % 3],
                          slot_sum(), slot_dyn() + 2);
        end_phase(3);
        frontier_n = prev_sum(2);
        ncols = vload(sh->dyn[(phase - 1) & 3] + 2);
      }
      if (ncols > 0) {  // in-hub columns: one more phase, chunks over the grid
        begin_phase();
        phase_activate_long<V>(p, frontier(tok + 1), ncols, slot_sum());
        end_phase(3);
        frontier_n += prev_sum(2);
      }
      ++tok;  // the next lift consumes it
      if (frontier_n == 0) break;  // every changed vertex has only top predecessors
    } else if (inplace) {
      ++tok;  // the pushed frontier is discarded (the dense lift clears both bitmaps)
    }

    // ---- lift round `round + 1`
    uint32_t* next = p.chg[round & 1];
    begin_phase();
    if (leader && p.timeout_ns && t_prev - t_start > p.timeout_ns) sh->stop = 1;
    // (right after a certificate apply, a Jacobi dense round lifts only the
    // player-1 light vertices the apply listed below top)
    phase_lift<V>(p, dense, frontier(tok), frontier(tok + 1), sh->fr_cnt[(tok + 2) % 3], next,
                  chg, slot_sum(), slot_dyn(), p.mode == kModeSweep,
                  dense && cert_now && p.mode != kModeSweep);
    end_phase(1);
    inplace = !dense || p.mode == kModeSweep;  // a sweep round needs no commit
    if (inplace) {
      pushed = prev_sum(2);
      pushed_long = vload(sh->dyn[(phase - 1) & 3] + 2);
    }
    ++(dense ? rounds_dense : rounds_sparse);
    ++round;
    changed = prev_sum(0);
  }

  stats_exit(p.ctr);
  if (leader) {
    if (sh->xerr) status = 7;
    p.ctr[kEpoch] = epoch;
    p.ctr[kRounds] = round;
    p.ctr[kDenseRounds] = rounds_dense;
    p.ctr[kSparseRounds] = rounds_sparse;
    p.ctr[kCertAttempts] = cert_attempts;
    p.ctr[kCertPasses] = cert_passes;
    p.ctr[kStatus] = status;
  }
}

}  // namespace EGS_FMT_NS
}  // namespace egs
