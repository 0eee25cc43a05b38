// test_solver_gpu.cpp — C++ parity tests of the drop-in, written against the
// REFERENCE API (proj/include/egsolve) the way the reference's own unit tests
// are (proj/tests/CMakeLists.txt:1-12 lists test_solver_seq / test_solver_par).
// Every check compares egsolve::solve_gpu with the reference solvers on the
// same arena: write_solution(make_solution(...)) bytes, W0/W1, and
// is_progress_measure; plus the error mapping.  Built by the Makefile into
// oracle/_ref/ (needs the reference headers), run on the GPU box by
// tests/test_cpp_dropin.py.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "egsolve/errors.hpp"
#include "egsolve/io.hpp"
#include "egsolve/measure_ops.hpp"
#include "egsolve/rng.hpp"
#include "egsolve/solver.hpp"
#include "solver_gpu.hpp"

using namespace egsolve;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond, what)                                                  \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      ++g_fail;                                                            \
      std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, what);   \
    }                                                                      \
  } while (0)

static int workers() {
  const unsigned hw = std::thread::hardware_concurrency();
  return hw ? (int)std::min(hw, 16u) : 1;
}

static void same_solution(const GameArena& a, Variant ref_variant, const char* what,
                          const GpuOptions& g = {}) {
  SolverOptions ro;
  ro.workers = ref_variant == Variant::kSeq ? 1 : workers();
  const SolveReport want = solve(a, ref_variant, ro);
  const SolveReport got = solve_gpu(a, SolverOptions{}, g);
  CHECK(got.measure.raw() == want.measure.raw(), what);
  CHECK(got.w0 == want.w0 && got.w1 == want.w1, what);
  CHECK(write_solution(make_solution(a, got)) == write_solution(make_solution(a, want)), what);
  CHECK(is_progress_measure(a, got.measure), what);
}

static GameArena fixed(uint64_t n, uint32_t d, int64_t W, uint64_t seed) {
  SplitMix64 r(seed);
  std::vector<Edge> e;
  std::vector<Owner> o(n);
  for (uint64_t v = 0; v < n; ++v) {
    o[v] = (v & 1) ? Owner::kPlayer1 : Owner::kPlayer0;
    for (uint32_t k = 0; k < d; ++k) {
      const VertexId dst = static_cast<VertexId>(r.next_below(n));
      e.push_back(Edge{static_cast<VertexId>(v), dst, r.next_in(-W, W)});
    }
  }
  return GameArena::build(static_cast<uint32_t>(n), e, o);
}

static GameArena random_arena(uint64_t seed, uint32_t max_n, uint32_t max_deg) {
  SplitMix64 r(seed);
  const uint32_t n = 1 + static_cast<uint32_t>(r.next_below(max_n));
  const int64_t Ws[] = {1, 2, 3, 10, 100, 1000, 1000000};
  const int64_t W = Ws[r.next_below(7)];
  std::vector<Edge> e;
  std::vector<Owner> o(n);
  for (uint32_t v = 0; v < n; ++v) {
    o[v] = r.next_below(2) ? Owner::kPlayer1 : Owner::kPlayer0;
    const uint32_t deg = 1 + static_cast<uint32_t>(r.next_below(max_deg));
    for (uint32_t k = 0; k < deg; ++k)
      e.push_back(Edge{v, static_cast<VertexId>(r.next_below(n)), r.next_in(-W, W)});
  }
  return GameArena::build(n, e, o);
}

int main() {
  // SPEC fixtures through the reference loader (io.hpp:19) and output format.
  const char* spec[][2] = {
      {"eg 2 2\nv 0 0\nv 1 1\ne 0 1 -1\ne 1 0 1\n", "0 1 1\n1 0\n"},           // G1
      {"eg 1 1\nv 0 0\ne 0 0 -1\n", "0 T\n"},                                   // P0 self-loop -1
      {"eg 1 1\nv 0 0\ne 0 0 0\n", "0 0 0\n"},                                  // self-loop 0
      {"eg 1 2\nv 0 0\ne 0 0 -1\ne 0 0 1\n", "0 0 0\n"},                        // P0 loops +-1
      {"eg 1 2\nv 0 1\ne 0 0 -1\ne 0 0 1\n", "0 T\n"},                          // P1 loops +-1
      {"eg 3 4\nv 0 0\nv 1 0\nv 2 0\ne 0 1 -5\ne 0 2 0\ne 1 1 0\ne 2 2 0\n",
       "0 0 2\n1 0 1\n2 0 2\n"},                                                // strategy example
  };
  for (auto& s : spec) {
    const GameArena a = parse_arena(s[0]);
    const SolveReport got = solve_any(a, kGpuVariant);
    CHECK(write_solution(make_solution(a, got)) == s[1], s[0]);
    same_solution(a, Variant::kSeq, s[0]);
  }
  // Random arenas: acceptance criterion 2 (byte-identical across solvers).
  for (uint64_t seed = 0; seed < 300; ++seed) {
    const GameArena a = random_arena(seed, 40, 6);
    same_solution(a, Variant::kSeq, "random arena vs solve_seq");
    GpuOptions dense, sparse, plain;
    dense.mode = EGS_MODE_DENSE;
    sparse.mode = EGS_MODE_SPARSE;
    plain.certify = false;
    if (seed % 3 == 0) same_solution(a, Variant::kSweep, "random dense", dense);
    if (seed % 3 == 1) same_solution(a, Variant::kFrontier, "random sparse", sparse);
    if (seed % 3 == 2) same_solution(a, Variant::kSweep, "random plain iteration", plain);
  }
  // Canonical shapes: C1 and 10^4 versions of C2/C4/C5.
  same_solution(fixed(10000, 4, 100, 1), Variant::kSweep, "C1");
  same_solution(fixed(10000, 8, 1000, 1), Variant::kSweep, "C2 shape");
  same_solution(fixed(10000, 16, 100, 1), Variant::kSweep, "C4 shape");
  same_solution(fixed(10000, 8, 100000, 1), Variant::kSweep, "C5 shape");
  // Device EPM verifier agrees with the reference's is_progress_measure.
  {
    const GameArena a = fixed(5000, 8, 1000, 3);
    SolverOptions ro;
    ro.workers = workers();
    const SolveReport r = solve(a, Variant::kSweep, ro);
    CHECK(is_progress_measure_gpu(a, r.measure), "epm on the least measure");
    std::vector<int64_t> bad = r.measure.raw();
    for (auto& x : bad)
      if (x != detail::kRawTop && x > 0) {
        x = 0;
        break;
      }
    const ProgressMeasure pb = ProgressMeasure::from_raw(bad, a.id());
    CHECK(is_progress_measure_gpu(a, pb) == is_progress_measure(a, pb), "epm on a broken measure");
  }
  // Error mapping: the round budget surfaces as the reference's exception.
  {
    const GameArena a = fixed(10000, 4, 100, 1);
    SolverOptions ro;
    ro.sweep_bound = 5;
    GpuOptions g;
    g.certify = false;
    bool thrown = false;
    try {
      solve_gpu(a, ro, g);
    } catch (const BoundExhaustedError&) {
      thrown = true;
    }
    CHECK(thrown, "BoundExhaustedError");
    SolverOptions bad;
    bad.workers = 0;
    thrown = false;
    try {
      solve_gpu(a, bad);
    } catch (const InvalidConfigError&) {
      thrown = true;
    }
    CHECK(thrown, "InvalidConfigError");
    // an explicit sweep_bound of 0 fails after the first raising round, as
    // in the reference (solver_par.cpp:149-150,184-188)
    SolverOptions zero;
    zero.sweep_bound = 0;
    thrown = false;
    try {
      solve(a, Variant::kSweep, zero);
    } catch (const BoundExhaustedError&) {
      thrown = true;
    }
    CHECK(thrown, "reference: sweep_bound = 0 -> BoundExhaustedError");
    thrown = false;
    try {
      solve_gpu(a, zero);
    } catch (const BoundExhaustedError&) {
      thrown = true;
    }
    CHECK(thrown, "gpu: sweep_bound = 0 -> BoundExhaustedError");
    // ... and an arena already at its fixpoint passes with sweep_bound = 0
    const GameArena calm = fixed(100, 2, 0, 1);
    CHECK(solve_gpu(calm, zero).measure.raw() == solve(calm, Variant::kSweep, zero).measure.raw(),
          "sweep_bound = 0 on a fixpoint");
    SolverOptions badmap;
    badmap.mapping = Mapping{Mapping::Kind::kChunked, 3};
    thrown = false;
    try {
      solve_gpu(a, badmap);
    } catch (const InvalidConfigError&) {
      thrown = true;
    }
    CHECK(thrown, "chunk 3 -> InvalidConfigError");
  }
  // The reference's usual options (workers = thread count, a chunked
  // mapping, debug checks) are accepted by the GPU entry point unchanged.
  {
    const GameArena a = fixed(10000, 8, 1000, 2);
    SolverOptions ro;
    ro.workers = 16;
    ro.mapping = Mapping{Mapping::Kind::kChunked, 8};
    ro.debug_checks = true;
    const SolveReport want = solve(a, Variant::kSweep, ro);
    const SolveReport got = solve_gpu(a, ro);
    CHECK(got.measure.raw() == want.measure.raw(), "workers = 16, chunked(8), debug_checks");
    CHECK(got.workers == 16 && got.mapping.kind == Mapping::Kind::kChunked, "report echoes options");
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
