"""ctypes binding of libegs_b200.so and the Python mirror of the reference API.

Every struct below mirrors ``include/egs_gpu.h`` field for field.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# EGS_LIB selects an alternative build of the same library (tuning experiments)
lib_path = os.environ.get("EGS_LIB") or os.path.join(_HERE, "libegs_b200.so")

if not os.path.exists(lib_path):  # no CPU fallback: the product is the CUDA library
    raise ImportError(
        f"{lib_path} is missing: build it with `make` (or __graft_entry__.build())"
    )
lib = C.CDLL(lib_path)

INT64_MAX = np.iinfo(np.int64).max

# --------------------------------------------------------------- errors ----
class EgsolveError(RuntimeError):
    """egsolve::Error (errors.hpp:11)."""


class InvalidConfigError(EgsolveError):
    """egsolve::InvalidConfigError (errors.hpp:75)."""


class TimeoutError_(EgsolveError):
    """egsolve::TimeoutError (errors.hpp:79)."""


class OverflowError_(EgsolveError):
    """egsolve::OverflowError (errors.hpp:34); also arenas outside the device
    representation (EGS_ERR_UNSUPPORTED)."""


class CudaError(EgsolveError):
    """Device failure (EGS_ERR_CUDA)."""


class BoundExhaustedError(EgsolveError):
    """egsolve::BoundExhaustedError (errors.hpp:67)."""


class InternalInvariantError(EgsolveError):
    """egsolve::InternalInvariantError (errors.hpp:83)."""


class InputError(EgsolveError):
    """Malformed arena input (EGS_ERR_INPUT): one of the loader errors below."""


class SyntaxError_(InputError):
    """egsolve::SyntaxError (errors.hpp:36): "line N: reason"."""


class CountMismatchError(InputError):
    """egsolve::CountMismatchError (errors.hpp:44)."""


class DanglingVertexIdError(InputError):
    """egsolve::DanglingVertexIdError (errors.hpp:24)."""


class NonTotalArenaError(InputError):
    """egsolve::NonTotalArenaError (errors.hpp:16)."""


_ERRORS = {
    1: InvalidConfigError,
    2: TimeoutError_,
    3: OverflowError_,
    4: CudaError,
    5: BoundExhaustedError,
    6: InternalInvariantError,
    7: InputError,
}
_INPUT_KINDS = {"SyntaxError": SyntaxError_, "CountMismatchError": CountMismatchError,
                "DanglingVertexIdError": DanglingVertexIdError,
                "NonTotalArenaError": NonTotalArenaError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib.egs_last_error().decode(errors="replace")
        cls = _ERRORS.get(rc, EgsolveError)
        if rc == 7:  # "<Kind>: <the reference's message>"
            kind, _, rest = msg.partition(": ")
            if kind in _INPUT_KINDS:
                cls, msg = _INPUT_KINDS[kind], rest
        raise cls(msg)


# -------------------------------------------------------------- structs ----
class ArenaView(C.Structure):
    _fields_ = [
        ("num_vertices", C.c_uint32),
        ("num_edges", C.c_uint64),
        ("csr_offsets", C.c_void_p),
        ("csr_targets", C.c_void_p),
        ("csr_weights", C.c_void_p),
        ("owners", C.c_void_p),
        ("credit_cap", C.c_int64),
        ("max_abs_weight", C.c_int64),
    ]


class GpuOpts(C.Structure):
    _fields_ = [
        ("n_gpus", C.c_int32),
        ("device", C.c_int32),
        ("certify", C.c_int32),
        ("cert_interval", C.c_int32),
        ("cert_growth", C.c_int32),
        ("sparse_div", C.c_int32),
        ("grid_ctas", C.c_int32),
        ("no_tma", C.c_int32),
        ("mode", C.c_int32),
        ("debug_checks", C.c_int32),
        ("timeout_seconds", C.c_double),
        ("round_bound", C.c_uint64),
        ("has_round_bound", C.c_int32),
        ("reserved_opts", C.c_int32),
    ]


_STAT_U64 = [
    "lifts", "applications", "pops", "rounds", "edges_relaxed", "witness_checks",
    "dense_rounds", "sparse_rounds", "cert_attempts", "cert_passes", "certified",
    "activations", "visits", "cert_rows", "cert_edges",
]
_STAT_F64 = [
    "upload_seconds", "solve_seconds", "download_seconds", "wall_seconds",
    "seed_seconds", "lift_seconds", "cert_seconds", "activate_seconds",
]


class GpuStats(C.Structure):
    _fields_ = (
        [(k, C.c_uint64) for k in _STAT_U64]
        + [(k, C.c_double) for k in _STAT_F64]
        + [("algo_bytes", C.c_uint64), ("lift_bytes", C.c_uint64),
           ("kernel_launches", C.c_uint64), ("value_bits", C.c_uint32),
           ("grid_ctas", C.c_uint32), ("lift_sub_seconds", C.c_double * 5),
           ("phase_detail_seconds", C.c_double * 5),
           ("edge_bytes", C.c_uint32), ("reserved0", C.c_uint32),
           ("algo_bytes_s8d", C.c_uint64), ("h2d_bytes", C.c_uint64)]
    )

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["lift_sub_seconds"] = list(self.lift_sub_seconds)
        d["phase_detail_seconds"] = list(self.phase_detail_seconds)
        return d


MAX_RANKS = 8


class PartPlan(C.Structure):
    """egs_part_plan (include/egs_gpu.h): the rank-major, class-balanced
    partition of the relabelled vertices."""
    _fields_ = [
        ("world", C.c_uint32), ("num_vertices", C.c_uint32),
        ("rank_lo", C.c_uint32 * (MAX_RANKS + 1)),
        ("class_lo", (C.c_uint32 * 7) * MAX_RANKS),
        ("piece", (C.c_uint32 * (MAX_RANKS + 1)) * 6),
        ("edges", C.c_uint64 * MAX_RANKS),
    ]

    def as_dict(self) -> dict:
        w = self.world
        return {"world": w, "num_vertices": self.num_vertices,
                "rank_lo": list(self.rank_lo)[:w + 1],
                "class_lo": [list(self.class_lo[r]) for r in range(w)],
                "piece": [list(self.piece[k])[:w + 1] for k in range(6)],
                "edges": list(self.edges)[:w]}


_P = C.c_void_p
IPC_HANDLE_BYTES = 128  # include/egs_gpu.h EGS_IPC_HANDLE_BYTES
lib.egs_part_plan_compute.argtypes = [C.POINTER(ArenaView), C.c_int32, C.POINTER(PartPlan)]
lib.egs_part_plan_compute.restype = C.c_int
lib.egs_part_create.argtypes = [C.POINTER(ArenaView), C.POINTER(GpuOpts), C.c_int32, C.c_int32,
                                C.POINTER(_P), C.POINTER(PartPlan), C.POINTER(GpuStats)]
lib.egs_part_create.restype = C.c_int
lib.egs_part_export.argtypes = [_P, C.c_char_p]
lib.egs_part_export.restype = C.c_int
lib.egs_part_connect.argtypes = [_P, C.c_char_p]
lib.egs_part_connect.restype = C.c_int
lib.egs_part_connect_local.argtypes = [C.POINTER(_P), C.c_int32]
lib.egs_part_connect_local.restype = C.c_int
lib.egs_part_solve.argtypes = [_P, C.POINTER(GpuStats)]
lib.egs_part_solve.restype = C.c_int
lib.egs_part_read_measure.argtypes = [_P, _P]
lib.egs_part_read_measure.restype = C.c_int
lib.egs_part_digest.argtypes = [_P, C.POINTER(C.c_uint64)]
lib.egs_part_digest.restype = C.c_int
lib.egs_part_destroy.argtypes = [_P]
lib.egs_part_destroy.restype = None
lib.egs_gpu_opts_default.argtypes = [C.POINTER(GpuOpts)]
lib.egs_gpu_solve.argtypes = [C.POINTER(ArenaView), C.POINTER(GpuOpts), _P, C.POINTER(GpuStats)]
lib.egs_gpu_solve.restype = C.c_int
lib.egs_ctx_create.argtypes = [C.POINTER(ArenaView), C.POINTER(GpuOpts), C.POINTER(_P), C.POINTER(GpuStats)]
lib.egs_ctx_create.restype = C.c_int
lib.egs_ctx_solve.argtypes = [_P, C.POINTER(GpuStats)]
lib.egs_ctx_solve.restype = C.c_int
lib.egs_ctx_read_measure.argtypes = [_P, _P]
lib.egs_ctx_read_measure.restype = C.c_int
lib.egs_ctx_is_progress_measure.argtypes = [_P, _P]
lib.egs_ctx_is_progress_measure.restype = C.c_int
lib.egs_ctx_write_solution.argtypes = [_P, _P, C.c_size_t]
lib.egs_ctx_write_solution.restype = C.c_int64
lib.egs_ctx_is_fixpoint.argtypes = [_P, _P]
lib.egs_ctx_is_fixpoint.restype = C.c_int
lib.egs_ctx_destroy.argtypes = [_P]
lib.egs_ctx_destroy.restype = None
lib.egs_write_solution.argtypes = [C.POINTER(ArenaView), _P, _P, C.c_size_t]
lib.egs_write_solution.restype = C.c_int64
lib.egs_host_arena_fixed.argtypes = [C.c_uint64, C.c_uint32, C.c_int64, C.c_uint64, C.c_int, C.POINTER(_P)]
lib.egs_host_arena_fixed.restype = C.c_int
lib.egs_host_arena_rmat.argtypes = [C.c_uint32, C.c_uint32, C.c_int64, C.c_uint64, C.c_int, C.POINTER(_P)]
lib.egs_host_arena_rmat.restype = C.c_int
lib.egs_host_arena_view.argtypes = [_P, C.POINTER(ArenaView)]
lib.egs_host_arena_view.restype = None
lib.egs_host_arena_free.argtypes = [_P]
lib.egs_host_arena_free.restype = None
lib.egs_host_arena_build.argtypes = [C.c_uint32, C.c_uint64, _P, _P, _P, _P, C.c_int,
                                     C.POINTER(_P)]
lib.egs_host_arena_build.restype = C.c_int
lib.egs_arena_parse_text.argtypes = [C.c_char_p, C.c_size_t, C.c_int, C.POINTER(_P)]
lib.egs_arena_parse_text.restype = C.c_int
lib.egs_arena_write_text.argtypes = [C.POINTER(ArenaView), _P, C.c_size_t]
lib.egs_arena_write_text.restype = C.c_int64
lib.egs_arena_save.argtypes = [C.POINTER(ArenaView), C.c_char_p]
lib.egs_arena_save.restype = C.c_int
lib.egs_arena_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(_P)]
lib.egs_arena_load.restype = C.c_int
lib.egs_host_alloc_pinned.argtypes = [C.c_size_t]
lib.egs_host_alloc_pinned.restype = _P
lib.egs_host_free_pinned.argtypes = [_P]
lib.egs_host_free_pinned.restype = None
lib.egs_last_error.restype = C.c_char_p
lib.egs_version.restype = C.c_char_p


# ---------------------------------------------------------------- arena ----
class GameArena:
    """Flattened ``egsolve::GameArena``: CSR rows in input order, owners and the
    cached ``ArenaStats`` fields the solve path needs (arena.hpp:24-31)."""

    def __init__(self, csr_offsets, csr_targets, csr_weights, owners,
                 credit_cap: int, max_abs_weight: int, _handle=None):
        self.csr_offsets = csr_offsets
        self.csr_targets = csr_targets
        self.csr_weights = csr_weights
        self.owners = owners
        self.credit_cap = int(credit_cap)
        self.max_abs_weight = int(max_abs_weight)
        self._handle = _handle

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h:
            lib.egs_host_arena_free(h)
            self._handle = None

    @property
    def num_vertices(self) -> int:
        return int(self.owners.shape[0])

    @property
    def num_edges(self) -> int:
        return int(self.csr_targets.shape[0])

    def is_player0(self, v: int) -> bool:
        return int(self.owners[v]) == 0

    def out_degree(self, v: int) -> int:
        return int(self.csr_offsets[v + 1] - self.csr_offsets[v])

    def view(self) -> ArenaView:
        return ArenaView(
            self.num_vertices, self.num_edges,
            self.csr_offsets.ctypes.data, self.csr_targets.ctypes.data,
            self.csr_weights.ctypes.data, self.owners.ctypes.data,
            self.credit_cap, self.max_abs_weight,
        )

    # --- construction ------------------------------------------------------
    @classmethod
    def _from_native(cls, handle) -> "GameArena":
        v = ArenaView()
        lib.egs_host_arena_view(handle, C.byref(v))
        n, m = v.num_vertices, v.num_edges

        def arr(ptr, count, ctype, dtype):
            if count == 0:
                return np.zeros(0, dtype=dtype)
            buf = (ctype * count).from_address(ptr)
            return np.frombuffer(buf, dtype=dtype, count=count)

        return cls(
            arr(v.csr_offsets, n + 1, C.c_uint64, np.uint64),
            arr(v.csr_targets, m, C.c_uint32, np.uint32),
            arr(v.csr_weights, m, C.c_int64, np.int64),
            arr(v.owners, n, C.c_uint8, np.uint8),
            v.credit_cap, v.max_abs_weight, _handle=handle,
        )

    @classmethod
    def fixed(cls, n: int, d: int, W: int, seed: int = 1, pinned: bool = False) -> "GameArena":
        """Canonical ``fixed(n, d, W, seed)`` arena."""
        h = _P()
        _check(lib.egs_host_arena_fixed(n, d, W, seed, int(pinned), C.byref(h)))
        return cls._from_native(h)

    @classmethod
    def rmat(cls, scale: int, edge_factor: int, W: int, seed: int = 1,
             pinned: bool = False) -> "GameArena":
        """Canonical ``rmat(scale, ef, W, seed)`` arena with sink fix."""
        h = _P()
        _check(lib.egs_host_arena_rmat(scale, edge_factor, W, seed, int(pinned), C.byref(h)))
        return cls._from_native(h)

    @classmethod
    def build(cls, num_vertices: int, edges, owners) -> "GameArena":
        """``GameArena::build`` (arena.cpp:17-78) through egs_host_arena_build:
        validation, stable CSR rows in input order, ``compute_stats``
        (arena.cpp:80-108) with its overflow headroom.  ``edges`` is an
        iterable of (src, dst, weight)."""
        n = int(num_vertices)
        edges = [tuple(int(x) for x in e) for e in edges]
        own = np.asarray(owners, dtype=np.int64).reshape(-1)
        if own.shape[0] != n:
            raise CountMismatchError("owner list does not cover every vertex")
        for s_, d_, w_ in edges:
            for x in (s_, d_):
                if not 0 <= x < n:
                    raise DanglingVertexIdError(f"edge references unknown vertex id {x}")
            if not (-(2 ** 63) < w_ < 2 ** 63):
                raise OverflowError_("edge weight magnitude not representable")
        src = np.ascontiguousarray([e[0] for e in edges], dtype=np.uint32)
        dst = np.ascontiguousarray([e[1] for e in edges], dtype=np.uint32)
        w = np.ascontiguousarray([e[2] for e in edges], dtype=np.int64)
        own8 = np.ascontiguousarray(own != 0, dtype=np.uint8)
        h = _P()
        _check(lib.egs_host_arena_build(n, len(edges), src.ctypes.data, dst.ctypes.data,
                                        w.ctypes.data, own8.ctypes.data, 0, C.byref(h)))
        return cls._from_native(h)

    @classmethod
    def parse(cls, text, pinned: bool = False) -> "GameArena":
        """``parse_arena`` (io.cpp:87-149) of the reference's text format,
        on every host thread (egs_arena_parse_text)."""
        data = text.encode() if isinstance(text, str) else bytes(text)
        h = _P()
        _check(lib.egs_arena_parse_text(data, len(data), int(pinned), C.byref(h)))
        return cls._from_native(h)

    @classmethod
    def load(cls, path: str, pinned: bool = False) -> "GameArena":
        """An arena saved by ``save`` (binary format, egs_arena_io.cpp)."""
        h = _P()
        _check(lib.egs_arena_load(os.fsencode(path), int(pinned), C.byref(h)))
        return cls._from_native(h)

    def save(self, path: str) -> None:
        v = self.view()
        _check(lib.egs_arena_save(C.byref(v), os.fsencode(path)))

    def write_text(self) -> str:
        """``write_arena`` (io.cpp:151-176), byte-identical."""
        v = self.view()
        n = lib.egs_arena_write_text(C.byref(v), None, 0)
        if n < 0:
            _check(int(-n))
        buf = C.create_string_buffer(max(int(n), 1))
        lib.egs_arena_write_text(C.byref(v), buf, n)
        return buf.raw[:n].decode()


# -------------------------------------------------------------- options ----
class Variant(enum.IntEnum):
    """egsolve::Variant (solver.hpp:16) plus the device variant."""
    SEQ = 0
    SWEEP = 1
    FRONTIER = 2
    GPU = 3


_MODES = {"auto": 0, "dense": 1, "sparse": 2, "sweep": 3}


@dataclass
class SolverOptions:
    """egsolve::SolverOptions (solver.hpp:33-42); ``workers`` counts GPUs."""
    workers: int = 1
    certify: bool = True
    cert_interval: int = 1
    cert_growth: int = 8
    sparse_div: int = 8
    grid_ctas: int = 0
    no_tma: bool = False
    mode: str = "auto"
    debug_checks: bool = False
    timeout_seconds: float = 0.0
    sweep_bound: Optional[int] = None
    device: int = -1

    def to_c(self) -> GpuOpts:
        if self.mode not in _MODES:
            raise InvalidConfigError(f"unknown mode {self.mode!r}")
        o = GpuOpts()
        lib.egs_gpu_opts_default(C.byref(o))
        o.n_gpus = int(self.workers)
        o.device = int(self.device)
        o.certify = int(bool(self.certify))
        o.cert_interval = int(self.cert_interval)
        o.cert_growth = int(self.cert_growth)
        o.sparse_div = int(self.sparse_div)
        o.grid_ctas = int(self.grid_ctas)
        o.no_tma = int(bool(self.no_tma) or os.environ.get("EGS_NO_TMA") == "1")
        o.mode = _MODES[self.mode]
        o.debug_checks = int(bool(self.debug_checks))
        o.timeout_seconds = float(self.timeout_seconds)
        # sweep_bound keeps the reference's optional semantics: None = default
        # budget, 0 = fail after the first round that raises something
        o.has_round_bound = int(self.sweep_bound is not None)
        o.round_bound = int(self.sweep_bound or 0)
        return o


class SolveReport:
    """egsolve::SolveReport (solver.hpp:47-59); ``measure`` is the raw int64
    encoding (INT64_MAX = top, energy.hpp:16).  ``w0`` / ``w1`` are the
    reference's winning_sets (measure_ops.cpp:43-54), computed on first use."""

    def __init__(self, measure: np.ndarray, lifts: int = 0, applications: int = 0,
                 pops: int = 0, rounds: int = 0, wall_seconds: float = 0.0,
                 variant: "Variant" = None, workers: int = 1, gpu: Optional[dict] = None):
        self.measure = measure
        self.lifts, self.applications, self.pops, self.rounds = lifts, applications, pops, rounds
        self.wall_seconds = wall_seconds
        self.variant = Variant.GPU if variant is None else variant
        self.workers = workers
        self.gpu = gpu or {}
        self._w = None

    def _sets(self):
        if self._w is None:
            top = self.measure == INT64_MAX
            self._w = (np.nonzero(~top)[0].astype(np.uint32), np.nonzero(top)[0].astype(np.uint32))
        return self._w

    @property
    def w0(self) -> np.ndarray:
        return self._sets()[0]

    @property
    def w1(self) -> np.ndarray:
        return self._sets()[1]


def _report(measure: np.ndarray, st: GpuStats, workers: int) -> SolveReport:
    return SolveReport(
        measure=measure, lifts=int(st.lifts), applications=int(st.applications),
        pops=int(st.pops), rounds=int(st.rounds), wall_seconds=float(st.wall_seconds),
        variant=Variant.GPU, workers=workers, gpu=st.as_dict(),
    )


def solve(arena: GameArena, variant: Variant = Variant.GPU,
          options: Optional[SolverOptions] = None,
          out: Optional[np.ndarray] = None) -> SolveReport:
    """``egsolve::solve`` (solver.hpp:86-87) for ``Variant.GPU``.  ``out``
    (int64[n], e.g. pinned via ``pinned_empty``) receives the measure."""
    if variant != Variant.GPU:
        raise InvalidConfigError("this library implements only the GPU variant")
    options = options or SolverOptions()
    opts = options.to_c()
    view = arena.view()
    if out is None:
        out = np.empty(arena.num_vertices, dtype=np.int64)
    elif out.dtype != np.int64 or out.shape != (arena.num_vertices,) or not out.flags.c_contiguous:
        raise InvalidConfigError("out must be a contiguous int64 array of num_vertices")
    st = GpuStats()
    _check(lib.egs_gpu_solve(C.byref(view), C.byref(opts), out.ctypes.data, C.byref(st)))
    return _report(out, st, options.workers)


class PinnedBuffer:
    """Page-locked host memory from egs_host_alloc_pinned (freed with the object)."""

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        self.ptr = lib.egs_host_alloc_pinned(max(self.nbytes, 1))
        if not self.ptr:
            raise CudaError("cudaMallocHost failed")

    def array(self, dtype, count: int) -> np.ndarray:
        buf = (C.c_uint8 * self.nbytes).from_address(self.ptr)
        return np.frombuffer(buf, dtype=dtype, count=count)

    def __del__(self):
        p = getattr(self, "ptr", None)
        if p:
            lib.egs_host_free_pinned(p)
            self.ptr = None


def pinned_empty(count: int, dtype=np.int64):
    """(array, owner): a page-locked numpy array; keep ``owner`` alive."""
    dt = np.dtype(dtype)
    pb = PinnedBuffer(count * dt.itemsize)
    return pb.array(dt, count), pb


def write_solution(arena: GameArena, measure) -> str:
    """``write_solution(make_solution(arena, report))`` (io.cpp:178-210)."""
    f = measure.measure if isinstance(measure, SolveReport) else measure
    f = np.ascontiguousarray(f, dtype=np.int64)
    view = arena.view()
    n = lib.egs_write_solution(C.byref(view), f.ctypes.data, None, 0)
    if n < 0:
        _check(int(-n))
    buf = C.create_string_buffer(int(n))
    lib.egs_write_solution(C.byref(view), f.ctypes.data, buf, n)
    return buf.raw[:n].decode()


class DeviceSolver:
    """Device-resident context (egs_ctx_*): upload once, solve many times."""

    def __init__(self, arena: GameArena, options: Optional[SolverOptions] = None):
        self.arena = arena
        self.options = options or SolverOptions()
        self._opts = self.options.to_c()
        self._view = arena.view()
        self._ctx = _P()
        self.upload_stats = GpuStats()
        _check(lib.egs_ctx_create(C.byref(self._view), C.byref(self._opts),
                                  C.byref(self._ctx), C.byref(self.upload_stats)))

    def solve(self) -> GpuStats:
        st = GpuStats()
        _check(lib.egs_ctx_solve(self._ctx, C.byref(st)))
        return st

    def read_measure(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.arena.num_vertices, dtype=np.int64)
        _check(lib.egs_ctx_read_measure(self._ctx, out.ctypes.data))
        return out

    def is_progress_measure(self, f: np.ndarray) -> bool:
        f = np.ascontiguousarray(f, dtype=np.int64)
        r = lib.egs_ctx_is_progress_measure(self._ctx, f.ctypes.data)
        if r < 0:
            _check(-r)
        return bool(r)

    def write_solution(self) -> str:
        """write_solution(make_solution(...)) of the solved measure, on the device."""
        n = lib.egs_ctx_write_solution(self._ctx, None, 0)
        if n < 0:
            _check(int(-n))
        buf = C.create_string_buffer(max(int(n), 1))
        r = lib.egs_ctx_write_solution(self._ctx, buf, n)
        if r < 0:
            _check(int(-r))
        return buf.raw[:n].decode()

    def is_fixpoint(self, f: np.ndarray) -> bool:
        """delta(f) == f everywhere (egs_ctx_is_fixpoint)."""
        f = np.ascontiguousarray(f, dtype=np.int64)
        r = lib.egs_ctx_is_fixpoint(self._ctx, f.ctypes.data)
        if r < 0:
            _check(-r)
        return bool(r)

    def close(self):
        if self._ctx:
            lib.egs_ctx_destroy(self._ctx)
            self._ctx = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
