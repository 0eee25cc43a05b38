// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" face over the compiled reference library (the
// /root/reference/proj sources, built by the Makefile into
// oracle/_ref/libegsolve_ref.so).  It lets the Python tests and bench.py's
// reference arm drive the UNMODIFIED reference solve path through its own
// public API: GameArena::build (arena.hpp:83-84), solve (solver.hpp:86-87),
// make_solution / write_solution (io.hpp:35-37), is_progress_measure
// (measure_ops.hpp:100).  The canonical generators use the reference's own
// SplitMix64 (rng.hpp) in the draw order of SURVEY.md Appendix B.
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "egsolve/io.hpp"
#include "egsolve/measure_ops.hpp"
#include "egsolve/rng.hpp"
#include "egsolve/solver.hpp"

using namespace egsolve;

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
  if (dynamic_cast<const TimeoutError*>(&e)) return 2;
  if (dynamic_cast<const OverflowError*>(&e)) return 3;
  if (dynamic_cast<const BoundExhaustedError*>(&e)) return 5;
  if (dynamic_cast<const InvalidConfigError*>(&e)) return 1;
  if (dynamic_cast<const InternalInvariantError*>(&e)) return 6;
  return 7;
}

template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

}  // namespace

extern "C" {

const char* egsref_last_error() { return g_err.c_str(); }

void* egsref_gen_fixed(uint64_t n, uint32_t d, int64_t W, uint64_t seed) {
  GameArena* out = nullptr;
  guarded([&] {
    SplitMix64 r(seed);
    std::vector<Edge> e;
    e.reserve(n * d);
    std::vector<Owner> o(n);
    for (uint64_t v = 0; v < n; ++v) {
      o[v] = (v & 1) ? Owner::kPlayer1 : Owner::kPlayer0;
      for (uint32_t k = 0; k < d; ++k) {
        VertexId dst = static_cast<VertexId>(r.next_below(n));
        int64_t w = r.next_in(-W, W);
        e.push_back(Edge{static_cast<VertexId>(v), dst, w});
      }
    }
    out = new GameArena(GameArena::build(static_cast<uint32_t>(n), e, o));
  });
  return out;
}

void* egsref_gen_rmat(uint32_t scale, uint32_t ef, int64_t W, uint64_t seed) {
  GameArena* out = nullptr;
  guarded([&] {
    SplitMix64 r(seed);
    const uint64_t n = 1ull << scale;
    std::vector<Edge> e;
    e.reserve(ef * n + n);
    std::vector<uint8_t> has_out(n, 0);
    for (uint64_t i = 0; i < (uint64_t)ef * n; ++i) {
      uint64_t u = 0, v = 0;
      for (uint32_t b = 0; b < scale; ++b) {
        double x = static_cast<double>(r.next() >> 11) * 0x1.0p-53;
        uint32_t q = x < 0.57 ? 0u : x < 0.76 ? 1u : x < 0.95 ? 2u : 3u;
        u = (u << 1) | (q >> 1);
        v = (v << 1) | (q & 1u);
      }
      int64_t w = r.next_in(-W, W);
      e.push_back(Edge{static_cast<VertexId>(u), static_cast<VertexId>(v), w});
      has_out[u] = 1;
    }
    std::vector<Owner> o(n);
    for (uint64_t v = 0; v < n; ++v) {
      o[v] = (v & 1) ? Owner::kPlayer1 : Owner::kPlayer0;
      if (!has_out[v]) {
        VertexId dst = static_cast<VertexId>(r.next_below(n));
        int64_t w = r.next_in(-W, W);
        e.push_back(Edge{static_cast<VertexId>(v), dst, w});
      }
    }
    out = new GameArena(GameArena::build(static_cast<uint32_t>(n), e, o));
  });
  return out;
}

// GameArena::build from a flat edge list (input order = row order).
void* egsref_build(uint32_t n, uint64_t m, const uint32_t* src,
                   const uint32_t* dst, const int64_t* w,
                   const uint8_t* owner) {
  GameArena* out = nullptr;
  guarded([&] {
    std::vector<Edge> e(m);
    for (uint64_t i = 0; i < m; ++i) e[i] = Edge{src[i], dst[i], w[i]};
    std::vector<Owner> o(n);
    for (uint32_t v = 0; v < n; ++v)
      o[v] = owner[v] ? Owner::kPlayer1 : Owner::kPlayer0;
    out = new GameArena(GameArena::build(n, e, o));
  });
  return out;
}

void egsref_free(void* a) { delete static_cast<GameArena*>(a); }

uint32_t egsref_num_vertices(void* a) {
  return static_cast<GameArena*>(a)->num_vertices();
}
uint64_t egsref_num_edges(void* a) {
  return static_cast<GameArena*>(a)->num_edges();
}
int64_t egsref_credit_cap(void* a) {
  return static_cast<GameArena*>(a)->stats().credit_cap;
}
int64_t egsref_max_abs_weight(void* a) {
  return static_cast<GameArena*>(a)->stats().max_abs_weight;
}

// Raw CSR spans of the built arena (arena.hpp:109-115).
void egsref_csr(void* a, const uint64_t** off, const uint32_t** dst,
                const int64_t** w, const uint8_t** owner) {
  auto* g = static_cast<GameArena*>(a);
  *off = g->csr_offsets().data();
  *dst = g->csr_targets().data();
  *w = g->csr_weights().data();
  *owner = reinterpret_cast<const uint8_t*>(g->owners().data());
}

// egsolve::solve (solver.hpp:86-87).  variant: 0 seq, 1 sweep, 2 frontier.
// chunk > 0 selects Mapping::chunked(chunk).  stats[6] = lifts, applications,
// pops, rounds, (unused), (unused); *wall = SolveReport::wall_seconds.
int egsref_solve(void* a, int variant, int workers, uint32_t chunk,
                 uint64_t sweep_bound, double timeout, int64_t* f_out,
                 uint64_t* stats, double* wall) {
  return guarded([&] {
    auto* g = static_cast<GameArena*>(a);
    SolverOptions opt;
    opt.workers = workers;
    if (chunk) opt.mapping = Mapping::chunked(chunk);
    if (sweep_bound) opt.sweep_bound = sweep_bound;
    opt.timeout_seconds = timeout;
    SolveReport rep = solve(*g, static_cast<Variant>(variant), opt);
    if (f_out)
      std::memcpy(f_out, rep.measure.raw().data(),
                  rep.measure.raw().size() * sizeof(int64_t));
    if (stats) {
      stats[0] = rep.lifts;
      stats[1] = rep.applications;
      stats[2] = rep.pops;
      stats[3] = rep.rounds;
    }
    if (wall) *wall = rep.wall_seconds;
  });
}

// write_solution(make_solution(arena, report)) for a given raw measure.
int64_t egsref_write_solution(void* a, const int64_t* f, char* buf,
                              size_t cap) {
  int64_t len = -1;
  int rc = guarded([&] {
    auto* g = static_cast<GameArena*>(a);
    SolveReport rep;
    rep.measure = ProgressMeasure::from_raw(
        std::vector<int64_t>(f, f + g->num_vertices()), g->id());
    std::string s = write_solution(make_solution(*g, rep));
    if (buf) std::memcpy(buf, s.data(), std::min(cap, s.size()));
    len = static_cast<int64_t>(s.size());
  });
  return rc ? -rc : len;
}

// parse_arena (io.hpp:19) of `text`: the arena, or nullptr with
// egsref_last_error() = "<Kind>: <what()>" for the loader's error types.
void* egsref_parse_arena(const char* text, size_t len) {
  GameArena* out = nullptr;
  try {
    out = new GameArena(parse_arena(std::string_view(text, len)));
  } catch (const SyntaxError& e) {
    g_err = std::string("SyntaxError: ") + e.what();
  } catch (const CountMismatchError& e) {
    g_err = std::string("CountMismatchError: ") + e.what();
  } catch (const DanglingVertexIdError& e) {
    g_err = std::string("DanglingVertexIdError: ") + e.what();
  } catch (const NonTotalArenaError& e) {
    g_err = std::string("NonTotalArenaError: ") + e.what();
  } catch (const OverflowError& e) {
    g_err = std::string("OverflowError: ") + e.what();
  } catch (const std::exception& e) {
    g_err = std::string("Error: ") + e.what();
  }
  return out;
}

int64_t egsref_write_arena(void* a, char* buf, size_t cap) {
  std::string s = write_arena(*static_cast<GameArena*>(a));
  if (buf) std::memcpy(buf, s.data(), std::min(cap, s.size()));
  return static_cast<int64_t>(s.size());
}

int egsref_is_progress_measure(void* a, const int64_t* f) {
  int r = -1;
  guarded([&] {
    auto* g = static_cast<GameArena*>(a);
    r = is_progress_measure(
            *g, ProgressMeasure::from_raw(
                    std::vector<int64_t>(f, f + g->num_vertices()), g->id()))
            ? 1
            : 0;
  });
  return r;
}

}  // extern "C"
