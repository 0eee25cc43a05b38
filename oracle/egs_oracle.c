/*
 * egs_oracle.c — TEST INFRASTRUCTURE ONLY (see egs_oracle.h).
 *
 * Plain-C restatement of the reference solve path.  Not linked by the product.
 */
#include "egs_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng -- */
/* SplitMix64::next (rng.hpp:19-25). */
uint64_t eo_splitmix64_next(uint64_t* s) {
  *s += 0x9E3779B97F4A7C15ULL;
  uint64_t z = *s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
/* next_below: plain modulo (rng.hpp:29). */
uint64_t eo_splitmix64_below(uint64_t* s, uint64_t n) {
  return eo_splitmix64_next(s) % n;
}
/* next_in: inclusive range (rng.hpp:32-36). */
int64_t eo_splitmix64_in(uint64_t* s, int64_t lo, int64_t hi) {
  uint64_t span = (uint64_t)hi - (uint64_t)lo + 1;
  return (int64_t)((uint64_t)lo + eo_splitmix64_below(s, span));
}

/* ---------------------------------------------------------------- arena -- */
void eo_arena_free(eo_arena* a) {
  if (!a) return;
  free(a->csr_off);
  free(a->csr_dst);
  free(a->csr_w);
  free(a->csc_off);
  free(a->csc_src);
  free(a->csc_w);
  free(a->owner);
  memset(a, 0, sizeof(*a));
}

/* compute_stats (arena.cpp:80-108): M_G = sum_v max(0, -min out-weight),
 * overflow-checked with headroom cap <= INT64_MAX - maxW - 2. */
static int compute_stats(eo_arena* g) {
  int64_t cap = 0, maxw = 0;
  uint32_t maxd = 0;
  for (uint32_t v = 0; v < g->n; ++v) {
    int64_t worst = 0;
    for (uint64_t i = g->csr_off[v]; i < g->csr_off[v + 1]; ++i) {
      int64_t w = g->csr_w[i];
      if (w < 0 && -w > worst) worst = -w;
      int64_t mag = w < 0 ? -w : w;
      if (mag > maxw) maxw = mag;
    }
    if (__builtin_add_overflow(cap, worst, &cap)) return EO_ERR_OVERFLOW;
    uint64_t deg = g->csr_off[v + 1] - g->csr_off[v];
    if (deg > maxd) maxd = (uint32_t)deg;
  }
  if (cap > INT64_MAX - maxw - 2) return EO_ERR_OVERFLOW;
  g->credit_cap = cap;
  g->max_abs_weight = maxw;
  g->max_out_degree = maxd;
  g->avg_out_degree = g->n == 0 ? 0.0 : (double)g->m / (double)g->n;
  return EO_OK;
}

/* GameArena::build (arena.cpp:17-78): validation, stable counting sort into
 * CSR rows (input order within a row), CSC as the stable transpose. */
int eo_arena_build(uint32_t n, uint64_t m, const uint32_t* src,
                   const uint32_t* dst, const int64_t* w, const uint8_t* owner,
                   eo_arena* out) {
  memset(out, 0, sizeof(*out));
  for (uint64_t i = 0; i < m; ++i) {
    if (src[i] >= n || dst[i] >= n) return EO_ERR_DANGLING;
    if (w[i] == INT64_MIN) return EO_ERR_OVERFLOW;
  }
  eo_arena g;
  memset(&g, 0, sizeof(g));
  g.n = n;
  g.m = m;
  g.owner = (uint8_t*)malloc(n ? n : 1);
  g.csr_off = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  g.csc_off = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  g.csr_dst = (uint32_t*)malloc((m ? m : 1) * sizeof(uint32_t));
  g.csr_w = (int64_t*)malloc((m ? m : 1) * sizeof(int64_t));
  g.csc_src = (uint32_t*)malloc((m ? m : 1) * sizeof(uint32_t));
  g.csc_w = (int64_t*)malloc((m ? m : 1) * sizeof(int64_t));
  uint64_t* cursor = (uint64_t*)malloc(((size_t)n + 1) * sizeof(uint64_t));
  if (!g.owner || !g.csr_off || !g.csc_off || !g.csr_dst || !g.csr_w ||
      !g.csc_src || !g.csc_w || !cursor) {
    free(cursor);
    eo_arena_free(&g);
    return EO_ERR_ALLOC;
  }
  for (uint32_t v = 0; v < n; ++v) g.owner[v] = owner[v] ? 1 : 0;
  for (uint64_t i = 0; i < m; ++i) g.csr_off[src[i] + 1]++;
  for (uint32_t v = 0; v < n; ++v) {
    if (g.csr_off[v + 1] == 0) { /* totality, arena.cpp:39 */
      free(cursor);
      eo_arena_free(&g);
      return EO_ERR_NON_TOTAL;
    }
    g.csr_off[v + 1] += g.csr_off[v];
  }
  memcpy(cursor, g.csr_off, (size_t)n * sizeof(uint64_t));
  for (uint64_t i = 0; i < m; ++i) {
    uint64_t slot = cursor[src[i]]++;
    g.csr_dst[slot] = dst[i];
    g.csr_w[slot] = w[i];
  }
  for (uint64_t i = 0; i < m; ++i) g.csc_off[g.csr_dst[i] + 1]++;
  for (uint32_t v = 0; v < n; ++v) g.csc_off[v + 1] += g.csc_off[v];
  memcpy(cursor, g.csc_off, (size_t)n * sizeof(uint64_t));
  for (uint32_t v = 0; v < n; ++v) {
    for (uint64_t i = g.csr_off[v]; i < g.csr_off[v + 1]; ++i) {
      uint64_t slot = cursor[g.csr_dst[i]]++;
      g.csc_src[slot] = v;
      g.csc_w[slot] = g.csr_w[i];
    }
  }
  free(cursor);
  int rc = compute_stats(&g);
  if (rc != EO_OK) {
    eo_arena_free(&g);
    return rc;
  }
  *out = g;
  return EO_OK;
}

/* ----------------------------------------------------------- generators -- */
/* fixed(n, d, W, seed) — SURVEY.md Appendix B: owners alternate (even = P0),
 * for v, for k<d: dst = next_below(n) then w = next_in(-W, W). */
int eo_gen_fixed(uint64_t n, uint32_t d, int64_t W, uint64_t seed,
                 eo_arena* out) {
  if (n < 1 || n > UINT32_MAX || d < 1 || W < 0) return EO_ERR_INVALID;
  uint64_t m = n * d;
  uint32_t* src = (uint32_t*)malloc(m * sizeof(uint32_t));
  uint32_t* dst = (uint32_t*)malloc(m * sizeof(uint32_t));
  int64_t* w = (int64_t*)malloc(m * sizeof(int64_t));
  uint8_t* own = (uint8_t*)malloc(n);
  if (!src || !dst || !w || !own) {
    free(src); free(dst); free(w); free(own);
    return EO_ERR_ALLOC;
  }
  uint64_t s = seed, e = 0;
  for (uint64_t v = 0; v < n; ++v) {
    own[v] = (uint8_t)(v & 1);
    for (uint32_t k = 0; k < d; ++k, ++e) {
      src[e] = (uint32_t)v;
      dst[e] = (uint32_t)eo_splitmix64_below(&s, n);
      w[e] = eo_splitmix64_in(&s, -W, W);
    }
  }
  int rc = eo_arena_build((uint32_t)n, m, src, dst, w, own, out);
  free(src); free(dst); free(w); free(own);
  return rc;
}

/* rmat(scale, ef, W, seed) — SURVEY.md Appendix B: Graph500 (a,b,c) =
 * (.57,.19,.19), unif() = (next() >> 11) * 2^-53, then one forced uniform
 * edge for every sink in ascending order; owners alternate. */
int eo_gen_rmat(uint32_t scale, uint32_t ef, int64_t W, uint64_t seed,
                eo_arena* out) {
  if (scale < 1 || scale > 31 || ef < 1 || W < 0) return EO_ERR_INVALID;
  uint64_t n = 1ULL << scale;
  uint64_t base = (uint64_t)ef * n;
  uint64_t cap = base + n;
  uint32_t* src = (uint32_t*)malloc(cap * sizeof(uint32_t));
  uint32_t* dst = (uint32_t*)malloc(cap * sizeof(uint32_t));
  int64_t* w = (int64_t*)malloc(cap * sizeof(int64_t));
  uint8_t* own = (uint8_t*)malloc(n);
  uint8_t* has_out = (uint8_t*)calloc(n, 1);
  if (!src || !dst || !w || !own || !has_out) {
    free(src); free(dst); free(w); free(own); free(has_out);
    return EO_ERR_ALLOC;
  }
  uint64_t s = seed, m = 0;
  const double k53 = 1.0 / 9007199254740992.0; /* 2^-53 */
  for (uint64_t i = 0; i < base; ++i) {
    uint64_t u = 0, v = 0;
    for (uint32_t b = 0; b < scale; ++b) {
      double r = (double)(eo_splitmix64_next(&s) >> 11) * k53;
      uint32_t q = r < 0.57 ? 0u : r < 0.76 ? 1u : r < 0.95 ? 2u : 3u;
      u = (u << 1) | (q >> 1);
      v = (v << 1) | (q & 1u);
    }
    src[m] = (uint32_t)u;
    dst[m] = (uint32_t)v;
    w[m] = eo_splitmix64_in(&s, -W, W);
    has_out[u] = 1;
    ++m;
  }
  for (uint64_t v = 0; v < n; ++v) {
    own[v] = (uint8_t)(v & 1);
    if (!has_out[v]) {
      src[m] = (uint32_t)v;
      dst[m] = (uint32_t)eo_splitmix64_below(&s, n);
      w[m] = eo_splitmix64_in(&s, -W, W);
      ++m;
    }
  }
  int rc = eo_arena_build((uint32_t)n, m, src, dst, w, own, out);
  free(src); free(dst); free(w); free(own); free(has_out);
  return rc;
}

/* ------------------------------------------------------------ measure ops -- */
/* raw_ominus (energy.hpp:20-31): top-absorbing truncated subtraction. The
 * overflow throws are unreachable for arenas that passed compute_stats. */
int64_t eo_raw_ominus(int64_t a, int64_t b) {
  if (a == EO_TOP) return EO_TOP;
  int64_t r;
  if (__builtin_sub_overflow(a, b, &r)) abort();
  if (r < 0) r = 0;
  if (r == EO_TOP) abort();
  return r;
}

/* raw_lift (measure_ops.hpp:32-52): P0 min with early exit at 0, P1 max with
 * early exit at top, then acc > credit_cap -> top (strictly greater). */
int64_t eo_raw_lift(const eo_arena* g, uint32_t v, const int64_t* f) {
  const uint64_t b = g->csr_off[v], e = g->csr_off[v + 1];
  int64_t acc = eo_raw_ominus(f[g->csr_dst[b]], g->csr_w[b]);
  if (g->owner[v] == 0) {
    for (uint64_t i = b + 1; i < e && acc > 0; ++i) {
      int64_t c = eo_raw_ominus(f[g->csr_dst[i]], g->csr_w[i]);
      if (c < acc) acc = c;
    }
  } else {
    for (uint64_t i = b + 1; i < e && acc != EO_TOP; ++i) {
      int64_t c = eo_raw_ominus(f[g->csr_dst[i]], g->csr_w[i]);
      if (c > acc) acc = c;
    }
  }
  return acc > g->credit_cap ? EO_TOP : acc;
}

/* satisfied_edge_count (solver_seq.cpp:57-65). */
static int64_t satisfied_edges(const eo_arena* g, const int64_t* f,
                               uint32_t v) {
  int64_t c = 0;
  const int64_t fv = f[v];
  for (uint64_t i = g->csr_off[v]; i < g->csr_off[v + 1]; ++i)
    if (fv >= eo_raw_ominus(f[g->csr_dst[i]], g->csr_w[i])) ++c;
  return c;
}

/* solve_seq (solver_seq.cpp:124-212). */
int eo_solve_seq(const eo_arena* g, int64_t* f, eo_stats* st) {
  const uint32_t n = g->n;
  const int64_t cap = g->credit_cap;
  memset(st, 0, sizeof(*st));
  if (n == 0) return EO_OK;
  int64_t* count = (int64_t*)calloc(n, sizeof(int64_t));
  uint8_t* in_list = (uint8_t*)calloc(n, 1);
  uint32_t* ring = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  if (!count || !in_list || !ring) {
    free(count); free(in_list); free(ring);
    return EO_ERR_ALLOC;
  }
  size_t head = 0, tail = 0, size = 0;
#define RQ_PUSH(x) do { ring[tail] = (x); tail = tail + 1 == n ? 0 : tail + 1; ++size; } while (0)
  for (uint32_t v = 0; v < n; ++v) f[v] = 0;
  /* seeding (solver_seq.cpp:136-154) */
  for (uint32_t v = 0; v < n; ++v) {
    uint64_t nonneg = 0, deg = g->csr_off[v + 1] - g->csr_off[v];
    for (uint64_t i = g->csr_off[v]; i < g->csr_off[v + 1]; ++i)
      if (g->csr_w[i] >= 0) ++nonneg;
    int seeded = g->owner[v] == 0 ? nonneg == 0 : nonneg < deg;
    if (seeded) {
      RQ_PUSH(v);
      in_list[v] = 1;
    }
    if (g->owner[v] == 0) count[v] = seeded ? 0 : (int64_t)nonneg;
  }
  /* FIFO loop (solver_seq.cpp:162-205) */
  while (size) {
    uint32_t v = ring[head];
    head = head + 1 == n ? 0 : head + 1;
    --size;
    in_list[v] = 0;
    st->pops++;
    const int64_t old = f[v];
    const int64_t lifted = eo_raw_lift(g, v, f);
    st->applications++;
    st->edges_relaxed += g->csr_off[v + 1] - g->csr_off[v];
    (void)cap;
    if (lifted == old) continue;
    f[v] = lifted;
    st->lifts++;
    if (g->owner[v] == 0) count[v] = satisfied_edges(g, f, v);
    for (uint64_t i = g->csc_off[v]; i < g->csc_off[v + 1]; ++i) {
      uint32_t u = g->csc_src[i];
      int64_t w = g->csc_w[i];
      if (f[u] >= eo_raw_ominus(lifted, w)) continue; /* guard :193 */
      if (g->owner[u] == 0) {
        if (f[u] >= eo_raw_ominus(old, w)) count[u]--;
        if (count[u] <= 0 && !in_list[u]) {
          RQ_PUSH(u);
          in_list[u] = 1;
        }
      } else if (!in_list[u]) {
        RQ_PUSH(u);
        in_list[u] = 1;
      }
    }
  }
#undef RQ_PUSH
  free(count); free(in_list); free(ring);
  return EO_OK;
}

/* default_sweep_budget (solver_par.cpp:94-98), saturating. */
static uint64_t default_budget(const eo_arena* g) {
  uint64_t per = (uint64_t)g->credit_cap + 1, r;
  if (__builtin_mul_overflow(g->m, per, &r)) return UINT64_MAX;
  return r == UINT64_MAX ? r : r + 1;
}

/* solve_sweep, one worker (solver_par.cpp:126-245): every sweep lifts all
 * vertices in id order and stores only if cand > old; stop after a sweep
 * without change. */
int eo_solve_sweep(const eo_arena* g, uint64_t bound, int64_t* f,
                   eo_stats* st) {
  memset(st, 0, sizeof(*st));
  const uint32_t n = g->n;
  if (n == 0) return EO_OK;
  for (uint32_t v = 0; v < n; ++v) f[v] = 0;
  const uint64_t budget = bound ? bound : default_budget(g);
  for (;;) {
    int changed = 0;
    for (uint32_t v = 0; v < n; ++v) {
      int64_t cand = eo_raw_lift(g, v, f);
      st->applications++;
      st->edges_relaxed += g->csr_off[v + 1] - g->csr_off[v];
      if (cand > f[v]) {
        f[v] = cand;
        st->lifts++;
        changed = 1;
      }
    }
    st->rounds++;
    if (!changed) break;
    if (st->rounds >= budget) return EO_ERR_BOUND;
  }
  return EO_OK;
}

/* solve_frontier, one worker (solver_par.cpp:247-435): seed = vertices
 * violating at f == 0 (:368-387); each round lifts the frontier in order with
 * in-place stores; a raised vertex activates all non-top predecessors once
 * (:402-410); the gather drops top vertices (:305-311). */
int eo_solve_frontier(const eo_arena* g, int64_t* f, eo_stats* st) {
  memset(st, 0, sizeof(*st));
  const uint32_t n = g->n;
  if (n == 0) return EO_OK;
  uint32_t* cur = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  uint32_t* nxt = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  uint8_t* in_next = (uint8_t*)calloc(n, 1);
  if (!cur || !nxt || !in_next) {
    free(cur); free(nxt); free(in_next);
    return EO_ERR_ALLOC;
  }
  for (uint32_t v = 0; v < n; ++v) f[v] = 0;
  size_t nn = 0, nc = 0;
  for (uint32_t v = 0; v < n; ++v) {
    int any_neg = 0, all_neg = 1;
    for (uint64_t i = g->csr_off[v]; i < g->csr_off[v + 1]; ++i) {
      if (g->csr_w[i] < 0) any_neg = 1; else all_neg = 0;
    }
    if (g->owner[v] == 0 ? all_neg : any_neg) nxt[nn++] = v;
  }
  for (;;) {
    /* gather_and_partition (:292-340) */
    nc = 0;
    for (size_t i = 0; i < nn; ++i) {
      uint32_t u = nxt[i];
      in_next[u] = 0;
      if (f[u] != EO_TOP) cur[nc++] = u;
    }
    nn = 0;
    if (nc == 0) break;
    for (size_t i = 0; i < nc; ++i) {
      uint32_t v = cur[i];
      int64_t old = f[v];
      int64_t cand = eo_raw_lift(g, v, f);
      st->applications++;
      st->edges_relaxed += g->csr_off[v + 1] - g->csr_off[v];
      if (cand <= old) continue;
      f[v] = cand;
      st->lifts++;
      for (uint64_t k = g->csc_off[v]; k < g->csc_off[v + 1]; ++k) {
        uint32_t u = g->csc_src[k];
        if (f[u] == EO_TOP) continue;
        if (!in_next[u]) {
          in_next[u] = 1;
          nxt[nn++] = u;
        }
      }
    }
    st->pops += nc;
    st->rounds++;
  }
  free(cur); free(nxt); free(in_next);
  return EO_OK;
}

/* epm_condition_holds (measure_ops.cpp:17-31). */
int eo_epm_condition_holds(const eo_arena* g, const int64_t* f, uint32_t v) {
  const int64_t fv = f[v];
  if (g->owner[v] == 0) {
    for (uint64_t i = g->csr_off[v]; i < g->csr_off[v + 1]; ++i)
      if (fv >= eo_raw_ominus(f[g->csr_dst[i]], g->csr_w[i])) return 1;
    return 0;
  }
  for (uint64_t i = g->csr_off[v]; i < g->csr_off[v + 1]; ++i)
    if (fv < eo_raw_ominus(f[g->csr_dst[i]], g->csr_w[i])) return 0;
  return 1;
}

/* is_progress_measure (measure_ops.cpp:33-41). */
int eo_is_progress_measure(const eo_arena* g, const int64_t* f) {
  for (uint32_t v = 0; v < g->n; ++v)
    if (!eo_epm_condition_holds(g, f, v)) return 0;
  return 1;
}

/* extract_strategy (measure_ops.cpp:56-80). */
int eo_extract_strategy(const eo_arena* g, const int64_t* f, uint64_t* ch) {
  for (uint32_t v = 0; v < g->n; ++v) {
    ch[v] = UINT64_MAX;
    if (g->owner[v] != 0 || f[v] == EO_TOP) continue;
    const int64_t fv = f[v];
    int found = 0;
    for (uint64_t i = g->csr_off[v]; i < g->csr_off[v + 1]; ++i) {
      if (fv >= eo_raw_ominus(f[g->csr_dst[i]], g->csr_w[i])) {
        ch[v] = i;
        found = 1;
        break;
      }
    }
    if (!found) return EO_ERR_NO_WITNESS;
  }
  return EO_OK;
}

/* ---------------------------------------------------------------- text io -- */
typedef struct {
  char* buf;
  size_t cap;
  size_t len;
} sink;

static void put(sink* s, const char* p, size_t k) {
  if (s->buf && s->len < s->cap) {
    size_t room = s->cap - s->len;
    memcpy(s->buf + s->len, p, k < room ? k : room);
  }
  s->len += k;
}
static void put_u(sink* s, uint64_t v) {
  char t[24];
  int k = 0;
  do {
    t[k++] = (char)('0' + v % 10);
    v /= 10;
  } while (v);
  char r[24];
  for (int i = 0; i < k; ++i) r[i] = t[k - 1 - i];
  put(s, r, (size_t)k);
}
static void put_i(sink* s, int64_t v) {
  if (v < 0) {
    put(s, "-", 1);
    put_u(s, (uint64_t)0 - (uint64_t)v);
  } else {
    put_u(s, (uint64_t)v);
  }
}

/* write_solution(make_solution(arena, report)) (io.cpp:178-210). */
int64_t eo_write_solution(const eo_arena* g, const int64_t* f, char* buf,
                          size_t cap) {
  uint64_t* ch = (uint64_t*)malloc(((size_t)g->n + 1) * sizeof(uint64_t));
  if (!ch) return -EO_ERR_ALLOC;
  int rc = eo_extract_strategy(g, f, ch);
  if (rc != EO_OK) {
    free(ch);
    return -rc;
  }
  sink s = {buf, cap, 0};
  for (uint32_t v = 0; v < g->n; ++v) {
    put_u(&s, v);
    put(&s, " ", 1);
    if (f[v] == EO_TOP) put(&s, "T", 1); else put_i(&s, f[v]);
    if (ch[v] != UINT64_MAX) {
      put(&s, " ", 1);
      put_u(&s, g->csr_dst[ch[v]]);
    }
    put(&s, "\n", 1);
  }
  free(ch);
  return (int64_t)s.len;
}

/* write_arena (io.cpp:151-176). */
int64_t eo_write_arena(const eo_arena* g, char* buf, size_t cap) {
  sink s = {buf, cap, 0};
  put(&s, "eg ", 3);
  put_u(&s, g->n);
  put(&s, " ", 1);
  put_u(&s, g->m);
  put(&s, "\n", 1);
  for (uint32_t v = 0; v < g->n; ++v) {
    put(&s, "v ", 2);
    put_u(&s, v);
    put(&s, g->owner[v] == 0 ? " 0\n" : " 1\n", 3);
  }
  for (uint32_t v = 0; v < g->n; ++v) {
    for (uint64_t i = g->csr_off[v]; i < g->csr_off[v + 1]; ++i) {
      put(&s, "e ", 2);
      put_u(&s, v);
      put(&s, " ", 1);
      put_u(&s, g->csr_dst[i]);
      put(&s, " ", 1);
      put_i(&s, g->csr_w[i]);
      put(&s, "\n", 1);
    }
  }
  return (int64_t)s.len;
}

uint64_t eo_fnv1a64(const void* data, size_t len) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ULL;
  for (size_t i = 0; i < len; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}
