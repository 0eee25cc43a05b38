// solver_gpu.hpp — the C++ drop-in a maintainer adds next to
// egsolve::solve (proj/include/egsolve/solver.hpp:86-87).
//
// It is compiled against the REFERENCE headers (proj/include) and linked with
// the reference library plus libegs_b200.so; it only flattens the GameArena
// spans into the C-ABI of include/egs_gpu.h and rebuilds a SolveReport with
// the reference's own winning_sets, exactly as finish_report does
// (proj/src/solver_par.cpp:100-112).  Error codes come back as the
// reference's exception types (errors.hpp:11-85).
#pragma once

#include <cstdint>

#include "egs_gpu.h"
#include "egsolve/solver.hpp"

namespace egsolve {

// Value of the GPU variant in the reference's Variant enum (solver.hpp:14);
// a maintainer adds `kGpu = 3` there and a `case` in solve()
// (solver_seq.cpp:233-244) that calls solve_gpu.
inline constexpr Variant kGpuVariant = static_cast<Variant>(3);

struct GpuOptions {
  int device = -1;         // CUDA ordinal, -1 = current
  bool certify = true;     // losing-region certificate (exact)
  int mode = EGS_MODE_AUTO;
};

// SolverOptions::workers (CPU threads in the reference) is reported back but
// does not select GPUs: this entry point drives one GPU (multi-GPU goes
// through egs_part_*, paper_1710_03647_b200.distributed).  sweep_bound
// (including an explicit 0), timeout_seconds and debug_checks keep their
// meaning.
SolveReport solve_gpu(const GameArena& arena, const SolverOptions& options = {},
                      const GpuOptions& gpu = {}, egs_gpu_stats* stats = nullptr);

// solve() with the GPU variant added: kGpuVariant -> solve_gpu, anything else
// -> the reference's own solve().
SolveReport solve_any(const GameArena& arena, Variant variant,
                      const SolverOptions& options = {});

// is_progress_measure (measure_ops.hpp:100) evaluated on the device.
bool is_progress_measure_gpu(const GameArena& arena, const ProgressMeasure& f,
                             const GpuOptions& gpu = {});

}  // namespace egsolve
