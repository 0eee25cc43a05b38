"""ctypes bindings of the TEST-ONLY checkers:

* ``Oracle``    — oracle/libegs_oracle.so, the plain-C restatement of the
                  reference solve path (oracle/egs_oracle.h).
* ``RefLib``    — oracle/_ref/libegsolve_ref.so, the reference sources compiled
                  unmodified plus a thin extern "C" shim (oracle/ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs load these.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "libegs_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libegsolve_ref.so")
INT64_MAX = np.iinfo(np.int64).max


class EoArena(C.Structure):
    _fields_ = [
        ("n", C.c_uint32),
        ("m", C.c_uint64),
        ("csr_off", C.POINTER(C.c_uint64)),
        ("csr_dst", C.POINTER(C.c_uint32)),
        ("csr_w", C.POINTER(C.c_int64)),
        ("csc_off", C.POINTER(C.c_uint64)),
        ("csc_src", C.POINTER(C.c_uint32)),
        ("csc_w", C.POINTER(C.c_int64)),
        ("owner", C.POINTER(C.c_uint8)),
        ("credit_cap", C.c_int64),
        ("max_abs_weight", C.c_int64),
        ("max_out_degree", C.c_uint32),
        ("avg_out_degree", C.c_double),
    ]


class EoStats(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in
                ("lifts", "applications", "pops", "rounds", "edges_relaxed")]


class OracleArena:
    """An arena built by the C restatement (GameArena::build, arena.cpp:17-78)."""

    def __init__(self, lib, a: EoArena):
        self._lib = lib
        self.a = a

    def __del__(self):
        try:
            self._lib.eo_arena_free(C.byref(self.a))
        except Exception:
            pass

    @property
    def n(self) -> int:
        return int(self.a.n)

    @property
    def m(self) -> int:
        return int(self.a.m)

    def csr(self):
        n, m = self.n, self.m
        off = np.ctypeslib.as_array(self.a.csr_off, shape=(n + 1,)).copy()
        dst = np.ctypeslib.as_array(self.a.csr_dst, shape=(max(m, 1),))[:m].copy()
        w = np.ctypeslib.as_array(self.a.csr_w, shape=(max(m, 1),))[:m].copy()
        own = np.ctypeslib.as_array(self.a.owner, shape=(max(n, 1),))[:n].copy()
        return off, dst, w, own


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make`")
        L = C.CDLL(path)
        self.L = L
        A = C.POINTER(EoArena)
        L.eo_splitmix64_next.argtypes = [C.POINTER(C.c_uint64)]
        L.eo_splitmix64_next.restype = C.c_uint64
        L.eo_arena_build.argtypes = [C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p, A]
        L.eo_arena_free.argtypes = [A]
        L.eo_gen_fixed.argtypes = [C.c_uint64, C.c_uint32, C.c_int64, C.c_uint64, A]
        L.eo_gen_rmat.argtypes = [C.c_uint32, C.c_uint32, C.c_int64, C.c_uint64, A]
        for fn in ("eo_solve_seq", "eo_solve_frontier"):
            getattr(L, fn).argtypes = [A, C.c_void_p, C.POINTER(EoStats)]
        L.eo_solve_sweep.argtypes = [A, C.c_uint64, C.c_void_p, C.POINTER(EoStats)]
        L.eo_is_progress_measure.argtypes = [A, C.c_void_p]
        L.eo_raw_lift.argtypes = [A, C.c_uint32, C.c_void_p]
        L.eo_raw_lift.restype = C.c_int64
        L.eo_write_solution.argtypes = [A, C.c_void_p, C.c_void_p, C.c_size_t]
        L.eo_write_solution.restype = C.c_int64
        L.eo_write_arena.argtypes = [A, C.c_void_p, C.c_size_t]
        L.eo_write_arena.restype = C.c_int64
        L.eo_fnv1a64.argtypes = [C.c_void_p, C.c_size_t]
        L.eo_fnv1a64.restype = C.c_uint64

    # -- arenas
    def build(self, n, edges, owners) -> OracleArena:
        edges = list(edges)
        src = np.array([e[0] for e in edges], dtype=np.uint32)
        dst = np.array([e[1] for e in edges], dtype=np.uint32)
        w = np.array([e[2] for e in edges], dtype=np.int64)
        own = np.array(owners, dtype=np.uint8)
        a = EoArena()
        rc = self.L.eo_arena_build(n, len(edges), src.ctypes.data, dst.ctypes.data,
                                   w.ctypes.data, own.ctypes.data, C.byref(a))
        if rc:
            raise ValueError(f"eo_arena_build failed: {rc}")
        return OracleArena(self.L, a)

    def fixed(self, n, d, W, seed=1) -> OracleArena:
        a = EoArena()
        rc = self.L.eo_gen_fixed(n, d, W, seed, C.byref(a))
        if rc:
            raise ValueError(f"eo_gen_fixed failed: {rc}")
        return OracleArena(self.L, a)

    def rmat(self, scale, ef, W, seed=1) -> OracleArena:
        a = EoArena()
        rc = self.L.eo_gen_rmat(scale, ef, W, seed, C.byref(a))
        if rc:
            raise ValueError(f"eo_gen_rmat failed: {rc}")
        return OracleArena(self.L, a)

    # -- solvers
    def _solve(self, fn, g: OracleArena, *extra):
        f = np.zeros(max(g.n, 1), dtype=np.int64)
        st = EoStats()
        rc = fn(C.byref(g.a), *extra, f.ctypes.data, C.byref(st))
        if rc:
            raise RuntimeError(f"oracle solve failed: {rc}")
        return f[: g.n], {k: getattr(st, k) for k, _ in EoStats._fields_}

    def solve_seq(self, g):
        return self._solve(self.L.eo_solve_seq, g)

    def solve_sweep(self, g, bound=0):
        return self._solve(self.L.eo_solve_sweep, g, bound)

    def solve_frontier(self, g):
        return self._solve(self.L.eo_solve_frontier, g)

    def is_progress_measure(self, g, f) -> bool:
        f = np.ascontiguousarray(f, dtype=np.int64)
        return bool(self.L.eo_is_progress_measure(C.byref(g.a), f.ctypes.data))

    def write_solution(self, g, f) -> str:
        f = np.ascontiguousarray(f, dtype=np.int64)
        n = self.L.eo_write_solution(C.byref(g.a), f.ctypes.data, None, 0)
        if n < 0:
            raise RuntimeError(f"no witness: {n}")
        buf = C.create_string_buffer(max(int(n), 1))
        self.L.eo_write_solution(C.byref(g.a), f.ctypes.data, buf, n)
        return buf.raw[:n].decode()

    def write_arena(self, g) -> str:
        n = self.L.eo_write_arena(C.byref(g.a), None, 0)
        buf = C.create_string_buffer(int(n))
        self.L.eo_write_arena(C.byref(g.a), buf, n)
        return buf.raw[:n].decode()

    def fnv1a64(self, data: bytes) -> int:
        return int(self.L.eo_fnv1a64(data, len(data)))


def fnv1a64(data: bytes) -> int:
    h = 0xCBF29CE484222325
    for b in data:
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


class RefArena:
    def __init__(self, lib, h):
        self._lib = lib
        self.h = h

    def __del__(self):
        try:
            self._lib.egsref_free(self.h)
        except Exception:
            pass

    @property
    def n(self) -> int:
        return int(self._lib.egsref_num_vertices(self.h))

    @property
    def m(self) -> int:
        return int(self._lib.egsref_num_edges(self.h))

    def csr(self):
        off = C.POINTER(C.c_uint64)()
        dst = C.POINTER(C.c_uint32)()
        w = C.POINTER(C.c_int64)()
        own = C.POINTER(C.c_uint8)()
        self._lib.egsref_csr(self.h, C.byref(off), C.byref(dst), C.byref(w), C.byref(own))
        n, m = self.n, self.m
        return (np.ctypeslib.as_array(off, shape=(n + 1,)).copy(),
                np.ctypeslib.as_array(dst, shape=(m,)).copy(),
                np.ctypeslib.as_array(w, shape=(m,)).copy(),
                np.ctypeslib.as_array(own, shape=(n,)).copy())


class RefLib:
    """The unmodified reference library behind oracle/ref_shim.cpp."""

    SEQ, SWEEP, FRONTIER = 0, 1, 2

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make ref` where /root/reference exists")
        L = C.CDLL(path)
        self.L = L
        P = C.c_void_p
        L.egsref_gen_fixed.argtypes = [C.c_uint64, C.c_uint32, C.c_int64, C.c_uint64]
        L.egsref_gen_fixed.restype = P
        L.egsref_gen_rmat.argtypes = [C.c_uint32, C.c_uint32, C.c_int64, C.c_uint64]
        L.egsref_gen_rmat.restype = P
        L.egsref_build.argtypes = [C.c_uint32, C.c_uint64, P, P, P, P]
        L.egsref_build.restype = P
        L.egsref_free.argtypes = [P]
        L.egsref_num_vertices.argtypes = [P]
        L.egsref_num_vertices.restype = C.c_uint32
        L.egsref_num_edges.argtypes = [P]
        L.egsref_num_edges.restype = C.c_uint64
        L.egsref_credit_cap.argtypes = [P]
        L.egsref_credit_cap.restype = C.c_int64
        L.egsref_max_abs_weight.argtypes = [P]
        L.egsref_max_abs_weight.restype = C.c_int64
        L.egsref_csr.argtypes = [P, P, P, P, P]
        L.egsref_solve.argtypes = [P, C.c_int, C.c_int, C.c_uint32, C.c_uint64, C.c_double,
                                   P, P, C.POINTER(C.c_double)]
        L.egsref_solve.restype = C.c_int
        L.egsref_write_solution.argtypes = [P, P, P, C.c_size_t]
        L.egsref_write_solution.restype = C.c_int64
        L.egsref_write_arena.argtypes = [P, P, C.c_size_t]
        L.egsref_write_arena.restype = C.c_int64
        L.egsref_is_progress_measure.argtypes = [P, P]
        L.egsref_is_progress_measure.restype = C.c_int
        L.egsref_last_error.restype = C.c_char_p
        L.egsref_parse_arena.argtypes = [C.c_char_p, C.c_size_t]
        L.egsref_parse_arena.restype = P

    def _wrap(self, h):
        if not h:
            raise RuntimeError(self.L.egsref_last_error().decode())
        return RefArena(self.L, h)

    def fixed(self, n, d, W, seed=1):
        return self._wrap(self.L.egsref_gen_fixed(n, d, W, seed))

    def rmat(self, scale, ef, W, seed=1):
        return self._wrap(self.L.egsref_gen_rmat(scale, ef, W, seed))

    def build(self, n, edges, owners):
        edges = list(edges)
        src = np.array([e[0] for e in edges], dtype=np.uint32)
        dst = np.array([e[1] for e in edges], dtype=np.uint32)
        w = np.array([e[2] for e in edges], dtype=np.int64)
        own = np.array(owners, dtype=np.uint8)
        return self._wrap(self.L.egsref_build(n, len(edges), src.ctypes.data, dst.ctypes.data,
                                              w.ctypes.data, own.ctypes.data))

    def parse_arena(self, text: bytes):
        """(arena, None) or (None, "<Kind>: <what()>") from parse_arena."""
        h = self.L.egsref_parse_arena(text, len(text))
        if not h:
            return None, self.L.egsref_last_error().decode()
        return RefArena(self.L, h), None

    def credit_cap(self, a) -> int:
        return int(self.L.egsref_credit_cap(a.h))

    def solve(self, a, variant=1, workers=1, chunk=0, sweep_bound=0, timeout=0.0):
        """Returns (measure, stats dict, wall_seconds); raises on error."""
        f = np.zeros(max(a.n, 1), dtype=np.int64)
        st = np.zeros(6, dtype=np.uint64)
        wall = C.c_double()
        rc = self.L.egsref_solve(a.h, variant, workers, chunk, sweep_bound, timeout,
                                 f.ctypes.data, st.ctypes.data, C.byref(wall))
        if rc:
            err = RuntimeError(self.L.egsref_last_error().decode())
            err.code = rc
            raise err
        return f[: a.n], dict(lifts=int(st[0]), applications=int(st[1]), pops=int(st[2]),
                              rounds=int(st[3])), wall.value

    def write_solution(self, a, f) -> str:
        f = np.ascontiguousarray(f, dtype=np.int64)
        n = self.L.egsref_write_solution(a.h, f.ctypes.data, None, 0)
        if n < 0:
            raise RuntimeError(self.L.egsref_last_error().decode())
        buf = C.create_string_buffer(max(int(n), 1))
        self.L.egsref_write_solution(a.h, f.ctypes.data, buf, n)
        return buf.raw[:n].decode()

    def write_arena(self, a) -> str:
        n = self.L.egsref_write_arena(a.h, None, 0)
        buf = C.create_string_buffer(int(n))
        self.L.egsref_write_arena(a.h, buf, n)
        return buf.raw[:n].decode()

    def is_progress_measure(self, a, f) -> bool:
        f = np.ascontiguousarray(f, dtype=np.int64)
        return self.L.egsref_is_progress_measure(a.h, f.ctypes.data) == 1
