// solver_gpu.cpp — see solver_gpu.hpp.
#include "solver_gpu.hpp"

#include <chrono>
#include <string>
#include <vector>

#include "egsolve/errors.hpp"
#include "egsolve/measure_ops.hpp"

namespace egsolve {
namespace {

egs_arena_view view_of(const GameArena& a) {
  egs_arena_view v{};
  v.num_vertices = a.num_vertices();
  v.num_edges = a.num_edges();
  v.csr_offsets = a.csr_offsets().data();
  v.csr_targets = a.csr_targets().data();
  v.csr_weights = a.csr_weights().data();
  static_assert(sizeof(Owner) == 1, "owners are passed as bytes");
  v.owners = reinterpret_cast<const uint8_t*>(a.owners().data());
  v.credit_cap = a.stats().credit_cap;
  v.max_abs_weight = a.stats().max_abs_weight;
  return v;
}

// The reference's validate_options (solver_par.cpp:41-51): the same
// InvalidConfigError for the same options, although neither the worker count
// nor the mapping changes what the device computes (results are identical
// for every mapping, SPEC.md acceptance criterion 9).
void validate_like_reference(const SolverOptions& o) {
  if (o.workers < 1 || o.workers > 1024)
    throw InvalidConfigError("worker count must be in [1, 1024]");
  if (o.mapping.kind == Mapping::Kind::kChunked) {
    const uint32_t h = o.mapping.chunk;
    if (h == 0 || h > 64 || (h & (h - 1)) != 0)
      throw InvalidConfigError("chunk size must be a power of two in [1, 64]");
  }
}

egs_gpu_opts opts_of(const SolverOptions& o, const GpuOptions& g) {
  egs_gpu_opts c;
  egs_gpu_opts_default(&c);
  // SolverOptions::workers counts CPU threads in the reference; this entry
  // point drives one GPU whatever it says (multi-GPU: egs_part_*)
  c.n_gpus = 1;
  c.device = g.device;
  c.certify = g.certify ? 1 : 0;
  c.mode = g.mode;
  c.debug_checks = o.debug_checks ? 1 : 0;
  c.timeout_seconds = o.timeout_seconds;
  c.has_round_bound = o.sweep_bound.has_value() ? 1 : 0;
  c.round_bound = o.sweep_bound.value_or(0);
  return c;
}

[[noreturn]] void rethrow(int rc) {
  const std::string msg = egs_last_error();
  switch (rc) {
    case EGS_ERR_INVALID_CONFIG: throw InvalidConfigError(msg);
    case EGS_ERR_TIMEOUT: throw TimeoutError(msg);
    case EGS_ERR_UNSUPPORTED: throw OverflowError(msg);
    case EGS_ERR_BOUND: throw BoundExhaustedError(msg);
    case EGS_ERR_INTERNAL: throw InternalInvariantError(msg);
    default: throw Error("device failure: " + msg);
  }
}

}  // namespace

SolveReport solve_gpu(const GameArena& arena, const SolverOptions& options,
                      const GpuOptions& gpu, egs_gpu_stats* stats) {
  const auto start = std::chrono::steady_clock::now();
  validate_like_reference(options);
  const egs_arena_view v = view_of(arena);
  const egs_gpu_opts o = opts_of(options, gpu);
  std::vector<int64_t> raw(arena.num_vertices());
  egs_gpu_stats st{};
  const int rc = egs_gpu_solve(&v, &o, raw.data(), &st);
  if (rc != EGS_OK) rethrow(rc);
  if (stats) *stats = st;
  SolveReport report;
  report.measure = ProgressMeasure::from_raw(std::move(raw), arena.id());
  std::tie(report.w0, report.w1) = winning_sets(report.measure);
  report.lifts = st.lifts;
  report.applications = st.applications;
  report.pops = st.pops;
  report.rounds = st.rounds;
  report.variant = kGpuVariant;
  report.workers = options.workers;
  report.mapping = options.mapping;
  report.wall_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
  return report;
}

SolveReport solve_any(const GameArena& arena, Variant variant, const SolverOptions& options) {
  if (variant == kGpuVariant) return solve_gpu(arena, options);
  return solve(arena, variant, options);
}

bool is_progress_measure_gpu(const GameArena& arena, const ProgressMeasure& f,
                             const GpuOptions& gpu) {
  const egs_arena_view v = view_of(arena);
  egs_gpu_opts o = opts_of(SolverOptions{}, gpu);
  egs_ctx* ctx = nullptr;
  int rc = egs_ctx_create(&v, &o, &ctx, nullptr);
  if (rc != EGS_OK) rethrow(rc);
  const int r = egs_ctx_is_progress_measure(ctx, f.raw().data());
  egs_ctx_destroy(ctx);
  if (r < 0) rethrow(-r);
  return r == 1;
}

}  // namespace egsolve
