"""Multi-GPU solve: one persistent kernel per rank, exchange on the device
(include/egs_gpu.h egs_part_*).

The reference has no distributed path (its ``workers`` are threads,
``solver_par.cpp:231-236``).  Here ``world`` ranks solve one arena together:

* **Partition** (``plan``): the relabelled vertex order is rank-major; every
  (owner, out-degree) class is split into ``world`` pieces balanced by
  out-edges (``edge_balanced_bounds``, ``solver_par.cpp:62-80``), so each rank
  gets an equal share of player-0 rows, player-1 rows and hubs.  A rank keeps
  only its own rows and the transpose of its own rows.
* **Exchange**: the measure and the changed / removal bitmaps are replicated.
  A rank writes every value it raises, and every bit it sets, into its own
  replica and into its peers' (NVLink peer stores through CUDA IPC mappings,
  or plain stores for ranks of one process); at each phase boundary the ranks
  meet at a device-side barrier that also sums their phase counts, so all of
  them take the same schedule decision.  The host launches once per rank and
  waits once: no per-round host round trip, no host-staged collective.
* **Plumbing**: ``torch.distributed`` (NCCL or gloo) only exchanges the
  128-byte export records (CUDA IPC handle + GPU UUID) before the solve and
  checks afterwards that every rank holds the same measure (an all-gather of
  a 64-bit digest computed on the device, egs_part_digest).

``solve_distributed`` is the one-process-per-GPU entry (torchrun);
``solve_local`` runs several ranks in ONE process (several GPUs, or several
ranks sharing one GPU -- the tests' way to run the device exchange on a
single-GPU box).  Both give the single-GPU solver's measure byte for byte.
"""
from __future__ import annotations

import ctypes as C
import threading
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as N


def plan(arena: N.GameArena, world: int) -> dict:
    """The partition of ``arena`` over ``world`` ranks (egs_part_plan_compute;
    host only, deterministic)."""
    pl = N.PartPlan()
    v = arena.view()
    N._check(N.lib.egs_part_plan_compute(C.byref(v), int(world), C.byref(pl)))
    return pl.as_dict()


class Partition:
    """This rank's context (egs_part_create): the arena relabelled by the
    plan, its own rows on ``options.device``."""

    def __init__(self, arena: N.GameArena, rank: int, world: int,
                 options: Optional[N.SolverOptions] = None):
        options = options or N.SolverOptions()
        opts = options.to_c()
        opts.n_gpus = int(world)
        self.arena, self.rank, self.world = arena, int(rank), int(world)
        self._view = arena.view()
        self._part = C.c_void_p()
        pl = N.PartPlan()
        st = N.GpuStats()
        N._check(N.lib.egs_part_create(C.byref(self._view), C.byref(opts), self.rank, self.world,
                                       C.byref(self._part), C.byref(pl), C.byref(st)))
        self.plan = pl.as_dict()
        self.upload_seconds = st.upload_seconds
        self.h2d_bytes = int(st.h2d_bytes)  # this rank's rows only (sharded upload)

    def export(self) -> bytes:
        buf = C.create_string_buffer(N.IPC_HANDLE_BYTES)
        N._check(N.lib.egs_part_export(self._part, buf))
        return buf.raw

    def connect(self, handles: Sequence[bytes]) -> None:
        """Map every peer's replicated state (handles[r] = rank r's export)."""
        blob = b"".join(h if i != self.rank else bytes(N.IPC_HANDLE_BYTES)
                        for i, h in enumerate(handles))
        N._check(N.lib.egs_part_connect(self._part, blob))

    @staticmethod
    def connect_local(parts: Sequence["Partition"]) -> None:
        arr = (C.c_void_p * len(parts))(*[p._part.value for p in parts])
        N._check(N.lib.egs_part_connect_local(arr, len(parts)))

    def solve(self) -> N.GpuStats:
        st = N.GpuStats()
        N._check(N.lib.egs_part_solve(self._part, C.byref(st)))
        return st

    def digest(self) -> int:
        """egs_part_digest: order-free 64-bit digest of this rank's replica."""
        d = C.c_uint64()
        N._check(N.lib.egs_part_digest(self._part, C.byref(d)))
        return int(d.value)

    def read_measure(self) -> np.ndarray:
        out = np.empty(self.arena.num_vertices, dtype=np.int64)
        N._check(N.lib.egs_part_read_measure(self._part, out.ctypes.data))
        return out

    def close(self):
        if self._part:
            N.lib.egs_part_destroy(self._part)
            self._part = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class PartitionReport:
    measure: np.ndarray
    rounds: int = 0
    wall_seconds: float = 0.0
    solve_seconds: float = 0.0          # device time of this rank's kernel
    edges_relaxed: int = 0              # this rank's
    edges_owned: int = 0                # out-edges of this rank's vertices (plan)
    h2d_bytes: int = 0                  # this rank's upload (own rows + vertex arrays)
    plan: dict = field(default_factory=dict)
    stats: dict = field(default_factory=dict)


class TorchComm:
    """The plumbing collectives over ``torch.distributed`` (any backend):
    an all-gather of small byte strings (IPC handles, digests)."""

    def __init__(self):
        import torch.distributed as dist

        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

    def allgather_bytes(self, b: bytes) -> list:
        out = [None] * self.world
        self.dist.all_gather_object(out, b)
        return out

    def barrier(self):
        self.dist.barrier()


def solve_distributed(arena: N.GameArena, options: Optional[N.SolverOptions] = None,
                      comm=None, part_factory=Partition, part=None) -> PartitionReport:
    """One process per GPU (torchrun): this rank's share of the solve.  Every
    rank returns the same measure (checked: all-gather of its SHA-256).
    ``part`` reuses a connected Partition (repeated solves)."""
    comm = comm or TorchComm()
    rank, world = comm.rank, comm.world
    t0 = time.perf_counter()
    if part is None:
        part = part_factory(arena, rank, world, options)
        if world > 1:
            part.connect(comm.allgather_bytes(part.export()))
        comm.barrier()
    st = part.solve()
    digests = comm.allgather_bytes(part.digest().to_bytes(8, "little"))
    if any(d != digests[0] for d in digests):
        raise N.InternalInvariantError("ranks disagree on the measure")
    f = part.read_measure()
    return PartitionReport(
        measure=f, rounds=int(st.rounds), wall_seconds=time.perf_counter() - t0,
        solve_seconds=float(st.solve_seconds), edges_relaxed=int(st.edges_relaxed),
        edges_owned=int(part.plan["edges"][rank]), h2d_bytes=part.h2d_bytes, plan=part.plan,
        stats=st.as_dict())


def solve_local(arena: N.GameArena, world: int, devices: Optional[Sequence[int]] = None,
                options: Optional[N.SolverOptions] = None, parts=None):
    """``world`` ranks in this process, one host thread each (``devices[r]``:
    rank r's GPU; default all on the current device).  Returns (reports,
    parts); pass ``parts`` back to solve again without a new upload."""
    import dataclasses

    options = options or N.SolverOptions()
    if parts is None:
        devices = list(devices) if devices is not None else [options.device] * world
        parts = [Partition(arena, r, world,
                           dataclasses.replace(options, device=devices[r], workers=world))
                 for r in range(world)]
        Partition.connect_local(parts)
    results: list = [None] * world
    errors: list = [None] * world

    def run(r):
        try:
            t0 = time.perf_counter()
            st = parts[r].solve()
            results[r] = (st, time.perf_counter() - t0)
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            errors[r] = e

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for e in errors:
        if e is not None:
            raise e
    reports = []
    for r in range(world):
        st, wall = results[r]
        reports.append(PartitionReport(
            measure=parts[r].read_measure(), rounds=int(st.rounds), wall_seconds=wall,
            solve_seconds=float(st.solve_seconds), edges_relaxed=int(st.edges_relaxed),
            edges_owned=int(parts[r].plan["edges"][r]), h2d_bytes=parts[r].h2d_bytes,
            plan=parts[r].plan, stats=st.as_dict()))
    return reports, parts
