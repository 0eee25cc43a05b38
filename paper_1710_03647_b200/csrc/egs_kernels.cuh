// egs_kernels.cuh — sm_100a kernels of the energy-game value-iteration path.
//
// Every kernel restates one step of the reference solve path
// (/root/reference/proj):
//   k_lift        raw_lift / raw_lift_chunked  measure_ops.hpp:32-83, applied
//                 as one synchronous (Jacobi) round of solve_frontier /
//                 solve_sweep  solver_par.cpp:205-228, 389-417
//   k_lift_heavy  the same lift, one CTA per high-degree row
//   k_activate    predecessor activation + dedup  solver_par.cpp:402-410
//   k_seed        seeding  solver_par.cpp:368-387, solver_seq.cpp:136-154
//   k_cert_*      losing-region certificate: proves vertices
//                 are in W1 so their value can jump straight to top.
//   k_epm         epm_condition_holds / is_progress_measure
//                 measure_ops.cpp:17-41
//
// Layout in HBM: CSR row offsets u32[n+1], packed edge records
// int2 {u32 dst, i32 w}[m], owner u8[n], CSC offsets u32[n+1] + sources
// u32[m]; measure V[n] x2 (ping-pong), player-0 witness edge int2[n].
#pragma once

#include <cstdint>

#include "egs_device.cuh"

namespace egs {

enum Counter : int {
  kLifts = 0,
  kApps = 1,
  kEdges = 2,
  kWitness = 3,
  kActScanned = 4,
  kCertified = 5,
  kPops = 6,
  kNumCounters = 8
};

struct DevArena {
  uint32_t n;
  uint32_t m;
  const uint32_t* off;    // n+1 CSR row offsets
  const int2* edge;       // m   {dst, w}
  const uint8_t* owner;   // n   0 = player 0
  const uint32_t* coff;   // n+1 CSC column offsets
  const uint32_t* csrc;   // m   predecessor ids
  int64_t cap;            // credit_cap (M_G)
};

template <class V>
struct LiftArgs {
  DevArena g;
  const V* fcur;             // measure of the previous round (read only)
  V* fnxt;                   // dense: full next measure; sparse: staged values
  int2* wit;                 // player-0 witness edge
  const uint32_t* items;     // sparse: frontier list; dense: nullptr (0..n-1)
  const uint32_t* count_dev; // sparse: frontier size on device
  uint32_t count;            // dense: n
  uint32_t heavy_thresh;     // rows longer than this go to k_lift_heavy
  int dense;
  uint32_t* changed_list;
  uint32_t* changed_count;
  unsigned long long* ctr;
};

// ---------------------------------------------------------------- lift ----
// One Jacobi lift round over the light rows.  G lanes cooperate on a row
// (the paper's GPU-w mapping; raw_lift_chunked with h = G):
// consecutive lanes read consecutive 8-byte edge records (coalesced), gather
// f(t), and fold with a G-lane shuffle tree.  Player-0 vertices first test
// their witness edge (argmin of their last lift): while it is satisfied the
// lift is a no-op (values only rise), so the row is not read.
template <class V, int G>
__global__ void __launch_bounds__(256) k_lift(LiftArgs<V> a) {
  constexpr V TOP = Top<V>::v;
  const uint32_t lane = lane_id();
  const uint32_t gl = lane & (G - 1);
  const int leader = (int)(lane & ~(uint32_t)(G - 1));
  const uint32_t count = a.count_dev ? *a.count_dev : a.count;
  const uint32_t groups_total = gridDim.x * (blockDim.x / G);
  unsigned long long n_apps = 0, n_lifts = 0, n_edges = 0, n_wit = 0;

  for (uint32_t item0 = (blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) / G;
       item0 < count; item0 += groups_total) {
    const uint32_t item = item0 + lane / G;
    const bool act = item < count;
    uint32_t v = 0;
    if (act) v = a.items ? __ldg(a.items + item) : item;
    V old = 0;
    uint32_t b = 0, e = 0;
    bool p0 = false, light = false, work = false;
    if (act) {
      old = a.fcur[v];
      b = __ldg(a.g.off + v);
      e = __ldg(a.g.off + v + 1);
      light = (e - b) <= a.heavy_thresh;
      p0 = __ldg(a.g.owner + v) == 0;
      work = light && old != TOP;
    }
    bool wsat = false;
    if (work && p0 && gl == 0) {
      const int2 we = a.wit[v];
      wsat = old >= ominus_cap<V>(a.fcur[we.x], we.y, a.g.cap);
    }
    wsat = __shfl_sync(0xffffffffu, wsat, leader);
    if (wsat) {
      work = false;
      if (gl == 0) ++n_wit;
    }
    V acc = p0 ? TOP : V(0);
    uint32_t bi = 0xFFFFFFFFu;
    if (work) {
      for (uint32_t i = b + gl; i < e; i += G) {
        const int2 ed = __ldg(a.g.edge + i);
        const V c = ominus_cap<V>(a.fcur[ed.x], ed.y, a.g.cap);
        if (p0) {
          if (c < acc) {
            acc = c;
            bi = i;
          }
        } else {
          acc = c > acc ? c : acc;
        }
      }
    }
    const V best = group_minmax<G>(acc, p0);
    uint32_t bsel = (p0 && acc == best) ? bi : 0xFFFFFFFFu;
    bsel = group_minmax<G>(bsel, true);
    bool changed = false;
    if (act && gl == 0 && light) {
      if (work) {
        ++n_apps;
        n_edges += e - b;
        const V nv = best > old ? best : old;  // clamped store (solver_par.cpp:399)
        changed = nv > old;
        if (changed) ++n_lifts;
        if (a.dense || changed) a.fnxt[v] = nv;
        if (p0 && bsel != 0xFFFFFFFFu) a.wit[v] = __ldg(a.g.edge + bsel);
      } else if (a.dense) {
        a.fnxt[v] = old;
      }
    }
    warp_append(changed, v, a.changed_list, a.changed_count);
  }
  warp_add_u64(n_apps, a.ctr + kApps);
  warp_add_u64(n_lifts, a.ctr + kLifts);
  warp_add_u64(n_edges, a.ctr + kEdges);
  warp_add_u64(n_wit, a.ctr + kWitness);
}

// Block-wide min/max with first-index tie break for player 0.
template <class V>
__device__ __forceinline__ void block_reduce_arg(V& val, uint32_t& idx,
                                                 bool is_min, V* s_val,
                                                 uint32_t* s_idx) {
  const uint32_t lane = lane_id();
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t nwarps = blockDim.x >> 5;
  V w = group_minmax<32>(val, is_min);
  uint32_t wi = (val == w) ? idx : 0xFFFFFFFFu;
  wi = group_minmax<32>(wi, true);
  if (lane == 0) {
    s_val[warp] = w;
    s_idx[warp] = wi;
  }
  __syncthreads();
  if (warp == 0) {
    V x = lane < nwarps ? s_val[lane] : (is_min ? Top<V>::v : V(0));
    uint32_t xi = lane < nwarps ? s_idx[lane] : 0xFFFFFFFFu;
    V r = group_minmax<32>(x, is_min);
    uint32_t ri = (x == r) ? xi : 0xFFFFFFFFu;
    ri = group_minmax<32>(ri, true);
    if (lane == 0) {
      s_val[0] = r;
      s_idx[0] = ri;
    }
  }
  __syncthreads();
  val = s_val[0];
  idx = s_idx[0];
}

// The same lift for rows longer than heavy_thresh: one CTA per row, used for
// the R-MAT hubs (max out-degree 159,848 at scale 22).
template <class V>
__global__ void __launch_bounds__(512) k_lift_heavy(LiftArgs<V> a,
                                                    const uint32_t* heavy,
                                                    uint32_t nheavy,
                                                    const uint32_t* bm_cur) {
  constexpr V TOP = Top<V>::v;
  __shared__ V s_val[32];
  __shared__ uint32_t s_idx[32];
  __shared__ int s_flag;
  unsigned long long n_apps = 0, n_lifts = 0, n_edges = 0, n_wit = 0;
  for (uint32_t h = blockIdx.x; h < nheavy; h += gridDim.x) {
    const uint32_t v = heavy[h];
    if (!a.dense && !((bm_cur[v >> 5] >> (v & 31)) & 1u)) continue;
    const V old = a.fcur[v];
    if (old == TOP) {
      if (a.dense && threadIdx.x == 0) a.fnxt[v] = old;
      continue;
    }
    const uint32_t b = a.g.off[v], e = a.g.off[v + 1];
    const bool p0 = a.g.owner[v] == 0;
    if (p0) {
      if (threadIdx.x == 0) {
        const int2 we = a.wit[v];
        s_flag = old >= ominus_cap<V>(a.fcur[we.x], we.y, a.g.cap);
      }
      __syncthreads();
      const int sat = s_flag;
      __syncthreads();
      if (sat) {
        if (threadIdx.x == 0) {
          ++n_wit;
          if (a.dense) a.fnxt[v] = old;
        }
        continue;
      }
    }
    V acc = p0 ? TOP : V(0);
    uint32_t bi = 0xFFFFFFFFu;
    for (uint32_t i = b + threadIdx.x; i < e; i += blockDim.x) {
      const int2 ed = __ldg(a.g.edge + i);
      const V c = ominus_cap<V>(a.fcur[ed.x], ed.y, a.g.cap);
      if (p0) {
        if (c < acc) {
          acc = c;
          bi = i;
        }
      } else {
        acc = c > acc ? c : acc;
      }
    }
    block_reduce_arg<V>(acc, bi, p0, s_val, s_idx);
    if (threadIdx.x == 0) {
      ++n_apps;
      n_edges += e - b;
      const V nv = acc > old ? acc : old;
      const bool changed = nv > old;
      if (a.dense || changed) a.fnxt[v] = nv;
      if (p0 && bi != 0xFFFFFFFFu) a.wit[v] = a.g.edge[bi];
      if (changed) {
        ++n_lifts;
        a.changed_list[atomicAdd(a.changed_count, 1u)] = v;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (n_apps) atomicAdd(a.ctr + kApps, n_apps);
    if (n_lifts) atomicAdd(a.ctr + kLifts, n_lifts);
    if (n_edges) atomicAdd(a.ctr + kEdges, n_edges);
    if (n_wit) atomicAdd(a.ctr + kWitness, n_wit);
  }
}

// Sparse rounds stage new values in fnxt; commit them into the authoritative
// measure once every lift of the round has read fcur (Jacobi semantics).
template <class V>
__global__ void k_commit(V* fcur, const V* fnxt, const uint32_t* list,
                         const uint32_t* count) {
  const uint32_t c = *count;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < c;
       i += gridDim.x * blockDim.x) {
    const uint32_t v = list[i];
    fcur[v] = fnxt[v];
  }
}

// ------------------------------------------------------------ worklist ----
// Predecessor activation (solver_par.cpp:402-410): every non-top predecessor
// of a vertex raised in this round enters the next frontier once.  Dedup is
// an atomicOr on a bitmap; new members are compacted into the list with a
// warp ballot + popc prefix and one atomicAdd per warp.
template <class V, int G>
__global__ void __launch_bounds__(256)
    k_activate(DevArena g, const V* f, const uint32_t* changed,
               const uint32_t* changed_count, uint32_t* bm_nxt,
               uint32_t* fr_list, uint32_t* fr_count,
               unsigned long long* ctr) {
  constexpr V TOP = Top<V>::v;
  const uint32_t lane = lane_id();
  const uint32_t gl = lane & (G - 1);
  const uint32_t count = *changed_count;
  const uint32_t groups_total = gridDim.x * (blockDim.x / G);
  unsigned long long scanned = 0;
  for (uint32_t item0 = (blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) / G;
       item0 < count; item0 += groups_total) {
    const uint32_t item = item0 + lane / G;
    uint32_t b = 0, e = 0;
    if (item < count) {
      const uint32_t v = changed[item];
      b = g.coff[v];
      e = g.coff[v + 1];
    }
    for (uint32_t i = b + gl; i < e; i += G) {
      const uint32_t u = __ldg(g.csrc + i);
      ++scanned;
      bool add = false;
      if (f[u] != TOP) {
        const uint32_t bit = 1u << (u & 31);
        add = !(atomicOr(bm_nxt + (u >> 5), bit) & bit);
      }
      warp_append(add, u, fr_list, fr_count);
    }
  }
  warp_add_u64(scanned, ctr + kActScanned);
}

// ---------------------------------------------------------------- seed ----
// f = 0 everywhere; frontier = vertices violating their condition at f = 0:
// player 0 with only negative moves, player 1 with some negative move
// (solver_par.cpp:366-387).  The player-0 witness starts at the first
// non-negative edge (satisfied at f = 0), or edge 0 for seeded vertices.
template <class V, int G>
__global__ void __launch_bounds__(256)
    k_seed(DevArena g, V* f0, V* f1, int2* wit, uint32_t* bm, uint32_t* fr_list,
           uint32_t* fr_count) {
  const uint32_t lane = lane_id();
  const uint32_t gl = lane & (G - 1);
  const uint32_t groups_total = gridDim.x * (blockDim.x / G);
  for (uint32_t item0 = (blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) / G;
       item0 < g.n; item0 += groups_total) {
    const uint32_t v = item0 + lane / G;
    const bool act = v < g.n;
    uint32_t b = 0, e = 0;
    bool p0 = false;
    if (act) {
      b = g.off[v];
      e = g.off[v + 1];
      p0 = g.owner[v] == 0;
    }
    uint32_t first_nonneg = 0xFFFFFFFFu;
    bool any_neg = false;
    for (uint32_t i = b + gl; i < e; i += G) {
      const int w = g.edge[i].y;
      if (w < 0) {
        any_neg = true;
      } else if (first_nonneg == 0xFFFFFFFFu) {
        first_nonneg = i;
      }
    }
    first_nonneg = group_minmax<G>(first_nonneg, true);
    any_neg = group_any<G>(any_neg);
    bool seeded = false;
    if (act && gl == 0) {
      f0[v] = 0;
      f1[v] = 0;
      const bool all_neg = first_nonneg == 0xFFFFFFFFu;
      seeded = p0 ? all_neg : any_neg;
      wit[v] = g.edge[all_neg ? b : first_nonneg];
      if (seeded) atomicOr(bm + (v >> 5), 1u << (v & 31));
    }
    warp_append(seeded, v, fr_list, fr_count);
  }
}

// --------------------------------------------------------- certificate ----
// Losing-region certificate.  cand starts as every non-top
// vertex; a pass removes
//   player 0: v unless every edge (v,t) has t top, or t in cand and
//             f(v) < f(t) - w;
//   player 1: v unless some edge (v,t) has t top, or t in cand and
//             f(v) < f(t) - w.
// At the greatest fixpoint every edge inside the certified set under the
// player-1 choice has f(v) - f(t) + w <= -1, so every cycle player 0 can
// close there is negative and player 1 wins: the vertices are in W1 and
// their least measure is top.
template <class V>
__global__ void k_cert_init(const V* f, uint8_t* cand, uint32_t n) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += gridDim.x * blockDim.x)
    cand[v] = f[v] != Top<V>::v;
}

template <class V, int G>
__global__ void __launch_bounds__(256)
    k_cert_prune(DevArena g, const V* f, uint8_t* cand, uint32_t* removed) {
  constexpr V TOP = Top<V>::v;
  const uint32_t lane = lane_id();
  const uint32_t gl = lane & (G - 1);
  const uint32_t groups_total = gridDim.x * (blockDim.x / G);
  uint32_t n_removed = 0;
  for (uint32_t item0 = (blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) / G;
       item0 < g.n; item0 += groups_total) {
    const uint32_t v = item0 + lane / G;
    const bool c = v < g.n && cand[v];
    bool p0 = false;
    bool all_good = true, any_good = false;
    if (c) {
      p0 = g.owner[v] == 0;
      const int64_t fv = static_cast<int64_t>(f[v]);
      const uint32_t b = g.off[v], e = g.off[v + 1];
      for (uint32_t i = b + gl; i < e; i += G) {
        const int2 ed = __ldg(g.edge + i);
        const V ft = f[ed.x];
        const bool good =
            ft == TOP ||
            (cand[ed.x] && fv < static_cast<int64_t>(ft) - (int64_t)ed.y);
        all_good &= good;
        any_good |= good;
      }
    }
    all_good = group_all<G>(all_good);
    any_good = group_any<G>(any_good);
    if (c && gl == 0 && !(p0 ? all_good : any_good)) {
      cand[v] = 0;
      ++n_removed;
    }
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1)
    n_removed += __shfl_xor_sync(0xffffffffu, n_removed, s);
  if (lane == 0 && n_removed) atomicAdd(removed, n_removed);
}

// Certified vertices jump to top; they are appended to the changed list so a
// sparse next round activates their predecessors.
template <class V>
__global__ void k_cert_apply(V* f, const uint8_t* cand, uint32_t n,
                             uint32_t* changed_list, uint32_t* changed_count,
                             unsigned long long* ctr) {
  unsigned long long c = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t start = blockIdx.x * blockDim.x + threadIdx.x;
  // uniform trip count per warp for warp_append
  for (uint32_t base = start & ~31u; base < n; base += stride) {
    const uint32_t v = base + (threadIdx.x & 31u);
    bool hit = false;
    if (v < n && cand[v] && f[v] != Top<V>::v) {
      f[v] = Top<V>::v;
      hit = true;
      ++c;
    }
    warp_append(hit, v, changed_list, changed_count);
  }
  warp_add_u64(c, ctr + kCertified);
}

// ------------------------------------------------------------ helpers ----
template <class V>
__global__ void k_widen(const V* f, int64_t* out, uint32_t n) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += gridDim.x * blockDim.x) {
    const V x = f[v];
    out[v] = x == Top<V>::v ? INT64_MAX : static_cast<int64_t>(x);
  }
}

// Pack the reference CSR (u64 offsets, u32 targets, i64 weights) into the
// device layout; flags weights outside int32.
__global__ void k_pack(uint32_t n, uint64_t m, const uint64_t* off64,
                       const uint32_t* dst, const int64_t* w64, uint32_t* off,
                       int2* edge, uint32_t* indeg, int* bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t start = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (uint64_t i = start; i <= n; i += stride) off[i] = (uint32_t)off64[i];
  for (uint64_t i = start; i < m; i += stride) {
    const int64_t w = w64[i];
    if (w < -2147483647LL || w > 2147483647LL) atomicExch(bad, 1);
    const uint32_t t = dst[i];
    if (t >= n) atomicExch(bad, 2);
    edge[i] = make_int2((int)t, (int)w);
    atomicAdd(indeg + (t < n ? t : 0), 1u);
  }
}

// Device CSC build (the paper does this with CUSPARSE csr2csc,
// PAPER.md:524-530).  Order inside a column is irrelevant to the solver, so
// the scatter uses an atomic cursor rather than a stable sort.
template <int G>
__global__ void __launch_bounds__(256)
    k_csc_scatter(uint32_t n, const uint32_t* off, const int2* edge,
                  uint32_t* cursor, uint32_t* csrc) {
  const uint32_t lane = lane_id();
  const uint32_t gl = lane & (G - 1);
  const uint32_t groups_total = gridDim.x * (blockDim.x / G);
  for (uint32_t item0 = (blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) / G;
       item0 < n; item0 += groups_total) {
    const uint32_t v = item0 + lane / G;
    if (v >= n) continue;
    const uint32_t b = off[v], e = off[v + 1];
    for (uint32_t i = b + gl; i < e; i += G) {
      const uint32_t t = (uint32_t)edge[i].x;
      csrc[atomicAdd(cursor + t, 1u)] = v;
    }
  }
}

// epm_condition_holds over every vertex for a host-supplied int64 measure
// (raw encoding, INT64_MAX = top), uncapped ⊖ exactly as measure_ops.cpp:17-31.
// *bad_count counts violated vertices; *overflow flags raw_ominus overflow.
__global__ void k_epm(DevArena g, const int64_t* f, unsigned long long* bad,
                      int* overflow) {
  unsigned long long nb = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < g.n;
       v += gridDim.x * blockDim.x) {
    const int64_t fv = f[v];
    const bool p0 = g.owner[v] == 0;
    bool ok = !p0;
    for (uint32_t i = g.off[v]; i < g.off[v + 1]; ++i) {
      const int2 ed = g.edge[i];
      const int64_t ft = f[ed.x];
      int64_t c;
      if (ft == INT64_MAX) {
        c = INT64_MAX;
      } else {
        if (__builtin_expect(ed.y < 0 && ft > INT64_MAX + (int64_t)ed.y, 0)) {
          atomicExch(overflow, 1);
          c = INT64_MAX;
        } else {
          c = ft - ed.y;
          if (c < 0) c = 0;
        }
      }
      if (p0) {
        if (fv >= c) {
          ok = true;
          break;
        }
      } else if (fv < c) {
        ok = false;
        break;
      }
    }
    if (!ok) ++nb;
  }
  if (nb) atomicAdd(bad, nb);
}

}  // namespace egs
