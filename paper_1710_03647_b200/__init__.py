"""B200-native solver for the initial-credit problem of energy games.

Python face of ``libegs_b200.so`` (C-ABI in ``include/egs_gpu.h``).  It mirrors
the reference C++ interface of the solve path (/root/reference/proj):

* ``GameArena``       — the flattened CSR spans of ``egsolve::GameArena``
                        (proj/include/egsolve/arena.hpp:37-133).
* ``SolverOptions``   — ``egsolve::SolverOptions`` (solver.hpp:33-42) plus the
                        device knobs.
* ``SolveReport``     — ``egsolve::SolveReport`` (solver.hpp:47-59).
* ``solve``           — ``egsolve::solve(arena, Variant, options)``
                        (solver.hpp:86-87) for the GPU variant.
* ``write_solution``  — ``write_solution(make_solution(arena, report))``
                        (io.cpp:178-210).
* error classes       — the ``egsolve::Error`` hierarchy (errors.hpp:11-85).

There is no CPU fallback: importing this package fails loudly if the CUDA
library has not been built (``python -c 'import __graft_entry__ as g; g.build()'``).
"""
from __future__ import annotations

from ._native import (  # noqa: F401
    BoundExhaustedError,
    CountMismatchError,
    CudaError,
    DanglingVertexIdError,
    DeviceSolver,
    EgsolveError,
    GameArena,
    InputError,
    InternalInvariantError,
    InvalidConfigError,
    NonTotalArenaError,
    OverflowError_,
    PinnedBuffer,
    SolveReport,
    SolverOptions,
    SyntaxError_,
    TimeoutError_,
    Variant,
    lib,
    lib_path,
    pinned_empty,
    solve,
    write_solution,
)

__all__ = [
    "BoundExhaustedError",
    "CudaError",
    "DeviceSolver",
    "EgsolveError",
    "GameArena",
    "InternalInvariantError",
    "InvalidConfigError",
    "OverflowError_",
    "PinnedBuffer",
    "SolveReport",
    "SolverOptions",
    "TimeoutError_",
    "Variant",
    "lib",
    "lib_path",
    "pinned_empty",
    "solve",
    "write_solution",
]
