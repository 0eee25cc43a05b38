// egs_host.cpp — host half of the C-ABI: canonical synthetic arenas and the
// reference output format.
//
//   egs_host_arena_fixed / _rmat   the canonical generators of SURVEY.md §8d
//                                  (Appendix B), drawn from splitmix64
//                                  (proj/include/egsolve/rng.hpp:11-37) and
//                                  laid out exactly as GameArena::build
//                                  (proj/src/arena.cpp:17-78) lays out CSR
//                                  rows: input order within a row.
//   egs_write_solution             write_solution(make_solution(...))
//                                  (proj/src/io.cpp:178-210) with the
//                                  first-witness strategy of extract_strategy
//                                  (proj/src/measure_ops.cpp:56-80).
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "egs_gpu.h"
#include "egs_host_arena.h"

void egs_internal_set_error(const std::string& msg);

namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

// splitmix64 output for the state reached after `i` draws from `seed`
// (SplitMix64::next, rng.hpp:19-25): state_i = seed + i * gamma.
inline uint64_t mix_at(uint64_t seed, uint64_t i) {
  uint64_t z = seed + i * kGamma;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

inline int64_t draw_in(uint64_t r, int64_t lo, int64_t hi) {
  const uint64_t span = static_cast<uint64_t>(hi) - static_cast<uint64_t>(lo) + 1;
  return static_cast<int64_t>(static_cast<uint64_t>(lo) + r % span);
}

template <class T>
T* host_alloc(size_t count, bool pinned) {
  if (count == 0) count = 1;
  if (pinned) {
    void* p = nullptr;
    if (cudaMallocHost(&p, count * sizeof(T)) != cudaSuccess) return nullptr;
    return static_cast<T*>(p);
  }
  return static_cast<T*>(std::malloc(count * sizeof(T)));
}

template <class T>
void host_free(T* p, bool pinned) {
  if (!p) return;
  if (pinned)
    cudaFreeHost(p);
  else
    std::free(p);
}

template <class Fn>
void parallel_for(uint64_t count, Fn&& fn) {
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const uint64_t chunks = std::min<uint64_t>(hw, std::max<uint64_t>(1, count / 65536));
  if (chunks <= 1) {
    fn(0, count);
    return;
  }
  std::vector<std::thread> pool;
  for (uint64_t c = 0; c < chunks; ++c) {
    const uint64_t lo = count * c / chunks, hi = count * (c + 1) / chunks;
    pool.emplace_back([&fn, lo, hi] { fn(lo, hi); });
  }
  for (auto& t : pool) t.join();
}

}  // namespace

egs_host_arena* egs_internal_arena_alloc(uint32_t n, uint64_t m, bool pinned) {
  auto* a = new egs_host_arena();
  a->n = n;
  a->m = m;
  a->pinned = pinned;
  a->off = host_alloc<uint64_t>((size_t)n + 1, pinned);
  a->dst = host_alloc<uint32_t>(m, pinned);
  a->w = host_alloc<int64_t>(m, pinned);
  a->owner = host_alloc<uint8_t>(n, pinned);
  if (!a->off || !a->dst || !a->w || !a->owner) {
    egs_host_arena_free(a);
    return nullptr;
  }
  return a;
}

void egs_internal_arena_free(egs_host_arena* a) { egs_host_arena_free(a); }

// compute_stats (arena.cpp:80-108): M_G and max |w| with the same overflow
// checks and headroom.
int egs_internal_finish_stats(egs_host_arena* a) {
  std::vector<int64_t> worst((size_t)a->n, 0);
  std::atomic<int64_t> maxw_all{0};
  parallel_for(a->n, [&](uint64_t lo, uint64_t hi) {
    int64_t mw = 0;
    for (uint64_t v = lo; v < hi; ++v) {
      int64_t wv = 0;
      for (uint64_t i = a->off[v]; i < a->off[v + 1]; ++i) {
        const int64_t w = a->w[i];
        if (w < 0 && -w > wv) wv = -w;
        const int64_t mag = w < 0 ? -w : w;
        if (mag > mw) mw = mag;
      }
      worst[v] = wv;
    }
    int64_t cur = maxw_all.load();
    while (mw > cur && !maxw_all.compare_exchange_weak(cur, mw)) {
    }
  });
  int64_t cap = 0;
  const int64_t maxw = maxw_all.load();
  for (uint32_t v = 0; v < a->n; ++v) {
    if (a->off[v + 1] == a->off[v]) {
      egs_internal_set_error("NonTotalArenaError: vertex " + std::to_string(v) +
                             " has no outgoing edge");
      return EGS_ERR_INPUT;
    }
    if (__builtin_add_overflow(cap, worst[v], &cap)) {
      egs_internal_set_error("credit bound exceeds the representable range");
      return EGS_ERR_UNSUPPORTED;
    }
  }
  if (cap > INT64_MAX - maxw - 2) {
    egs_internal_set_error("credit bound exceeds the representable range");
    return EGS_ERR_UNSUPPORTED;
  }
  a->credit_cap = cap;
  a->max_abs_weight = maxw;
  return EGS_OK;
}

namespace {

inline void append_uint(std::string& out, uint64_t v) {
  char buf[24];
  auto r = std::to_chars(buf, buf + sizeof(buf), v);
  out.append(buf, static_cast<size_t>(r.ptr - buf));
}

inline int64_t raw_ominus(int64_t a, int64_t b) {
  if (a == INT64_MAX) return INT64_MAX;
  int64_t r;
  if (__builtin_sub_overflow(a, b, &r)) return INT64_MAX;  // unreachable for valid measures
  return r < 0 ? 0 : r;
}

}  // namespace

extern "C" {

// fixed(n, d, W, seed): for v, for k < d: dst = next_below(n), w = next_in(-W, W)
// (two draws per edge, so edge e uses draws 2e+1 and 2e+2).
int egs_host_arena_fixed(uint64_t n, uint32_t d, int64_t W, uint64_t seed,
                         int pinned, egs_host_arena** out) {
  if (n < 1 || n > 0xFFFFFFFFull || d < 1 || W < 0) {
    egs_internal_set_error("invalid fixed() spec");
    return EGS_ERR_INVALID_CONFIG;
  }
  const uint64_t m = n * d;
  egs_host_arena* a = egs_internal_arena_alloc((uint32_t)n, m, pinned != 0);
  if (!a) {
    egs_internal_set_error("host allocation failed");
    return EGS_ERR_CUDA;
  }
  parallel_for(n, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t v = lo; v < hi; ++v) {
      a->owner[v] = (uint8_t)(v & 1);
      a->off[v] = v * d;
      for (uint32_t k = 0; k < d; ++k) {
        const uint64_t e = v * d + k;
        a->dst[e] = (uint32_t)(mix_at(seed, 2 * e + 1) % n);
        a->w[e] = draw_in(mix_at(seed, 2 * e + 2), -W, W);
      }
    }
  });
  a->off[n] = m;
  int rc = egs_internal_finish_stats(a);
  if (rc != EGS_OK) {
    egs_host_arena_free(a);
    return rc;
  }
  *out = a;
  return EGS_OK;
}

// rmat(scale, ef, W, seed): ef*2^scale Graph500 draws (a,b,c = .57,.19,.19,
// unif = (next() >> 11) * 2^-53, scale draws + one weight draw per edge),
// then one forced uniform edge per sink in ascending order.  Rows keep draw
// order (stable counting sort by source, arena.cpp:43-54).
int egs_host_arena_rmat(uint32_t scale, uint32_t ef, int64_t W, uint64_t seed,
                        int pinned, egs_host_arena** out) {
  if (scale < 1 || scale > 31 || ef < 1 || W < 0) {
    egs_internal_set_error("invalid rmat() spec");
    return EGS_ERR_INVALID_CONFIG;
  }
  const uint64_t n = 1ull << scale;
  const uint64_t base = (uint64_t)ef * n;
  const uint64_t per = scale + 1;
  std::vector<uint32_t> src(base), dst(base);
  std::vector<int64_t> w(base);
  const double k53 = 1.0 / 9007199254740992.0;
  parallel_for(base, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t e = lo; e < hi; ++e) {
      uint64_t u = 0, v = 0;
      for (uint32_t b = 0; b < scale; ++b) {
        const double r = (double)(mix_at(seed, e * per + b + 1) >> 11) * k53;
        const uint32_t q = r < 0.57 ? 0u : r < 0.76 ? 1u : r < 0.95 ? 2u : 3u;
        u = (u << 1) | (q >> 1);
        v = (v << 1) | (q & 1u);
      }
      src[e] = (uint32_t)u;
      dst[e] = (uint32_t)v;
      w[e] = draw_in(mix_at(seed, e * per + scale + 1), -W, W);
    }
  });
  std::vector<uint64_t> deg(n + 1, 0);
  for (uint64_t e = 0; e < base; ++e) deg[src[e]]++;
  uint64_t sinks = 0;
  for (uint64_t v = 0; v < n; ++v) sinks += deg[v] == 0;
  const uint64_t m = base + sinks;
  egs_host_arena* a = egs_internal_arena_alloc((uint32_t)n, m, pinned != 0);
  if (!a) {
    egs_internal_set_error("host allocation failed");
    return EGS_ERR_CUDA;
  }
  // sink edges continue the same stream: two draws each, ascending v
  uint64_t draw = base * per;
  std::vector<uint32_t> sink_dst;
  std::vector<int64_t> sink_w;
  sink_dst.reserve(sinks);
  sink_w.reserve(sinks);
  for (uint64_t v = 0; v < n; ++v) {
    if (deg[v] == 0) {
      sink_dst.push_back((uint32_t)(mix_at(seed, ++draw) % n));
      sink_w.push_back(draw_in(mix_at(seed, ++draw), -W, W));
      deg[v] = 1;
    }
  }
  a->off[0] = 0;
  for (uint64_t v = 0; v < n; ++v) {
    a->owner[v] = (uint8_t)(v & 1);
    a->off[v + 1] = a->off[v] + deg[v];
  }
  std::vector<uint64_t> cursor(a->off, a->off + n);
  for (uint64_t e = 0; e < base; ++e) {
    const uint64_t slot = cursor[src[e]]++;
    a->dst[slot] = dst[e];
    a->w[slot] = w[e];
  }
  uint64_t k = 0;
  for (uint64_t v = 0; v < n; ++v) {
    if (cursor[v] < a->off[v + 1]) {  // the forced sink edge
      a->dst[cursor[v]] = sink_dst[k];
      a->w[cursor[v]] = sink_w[k];
      ++k;
    }
  }
  int rc = egs_internal_finish_stats(a);
  if (rc != EGS_OK) {
    egs_host_arena_free(a);
    return rc;
  }
  *out = a;
  return EGS_OK;
}

void egs_host_arena_view(const egs_host_arena* a, egs_arena_view* v) {
  v->num_vertices = a->n;
  v->num_edges = a->m;
  v->csr_offsets = a->off;
  v->csr_targets = a->dst;
  v->csr_weights = a->w;
  v->owners = a->owner;
  v->credit_cap = a->credit_cap;
  v->max_abs_weight = a->max_abs_weight;
}

void egs_host_arena_free(egs_host_arena* a) {
  if (!a) return;
  host_free(a->off, a->pinned);
  host_free(a->dst, a->pinned);
  host_free(a->w, a->pinned);
  host_free(a->owner, a->pinned);
  delete a;
}

int64_t egs_write_solution(const egs_arena_view* g, const int64_t* f,
                           char* buf, size_t cap) {
  std::string out;
  out.reserve((size_t)g->num_vertices * 10);
  for (uint32_t v = 0; v < g->num_vertices; ++v) {
    append_uint(out, v);
    out += ' ';
    const int64_t fv = f[v];
    if (fv == INT64_MAX) {
      out += 'T';
    } else {
      append_uint(out, (uint64_t)fv);
    }
    if (g->owners[v] == 0 && fv != INT64_MAX) {
      bool found = false;
      for (uint64_t i = g->csr_offsets[v]; i < g->csr_offsets[v + 1]; ++i) {
        const uint32_t t = g->csr_targets[i];
        if (fv >= raw_ominus(f[t], g->csr_weights[i])) {
          out += ' ';
          append_uint(out, t);
          found = true;
          break;
        }
      }
      if (!found) {
        egs_internal_set_error("no witness successor at vertex " + std::to_string(v));
        return -EGS_ERR_INTERNAL;
      }
    }
    out += '\n';
  }
  if (buf) std::memcpy(buf, out.data(), std::min(cap, out.size()));
  return (int64_t)out.size();
}

const char* egs_version(void) { return "egs_b200 0.1 (sm_100a)"; }

}  // extern "C"
