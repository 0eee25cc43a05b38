"""Multi-GPU solve: vertex-range partition, one process per GPU.

The reference has no distributed path (its ``workers`` are threads,
``solver_par.cpp:231-236``).  Here every rank holds the whole arena (3 GB at
C4 against 180 GB of HBM) and a replica of the measure, lifts only its own
range of relabelled vertices, and after each step the ranks all-gather the
owned slices of the replicated array that step wrote.  Rounds are synchronous
(Jacobi), so the partitioned iteration is, round for round, the single-GPU
dense iteration of ``k_solve``; termination is a round that raises nothing
on any rank (one all-reduce), exactly the reference's ``changed`` latch
(``solver_par.cpp:170-194``).

Two pluggable pieces:

* ``DeviceSteps`` -- this rank's GPU through the C-ABI partition entry points
  (``egs_part_*`` in include/egs_gpu.h).  The replicated arrays are the
  library's own device buffers, wrapped (no copy) as torch tensors through
  ``__cuda_array_interface__`` so NCCL all-gathers them in place.
* ``TorchComm`` -- the collectives: ``torch.distributed`` over NCCL with
  device tensors (the product), or over gloo with host staging (the CPU and
  single-GPU tests of this orchestration).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N

STEP_ROUND1, STEP_LIFT, STEP_COMMIT, STEP_CERT_INIT, STEP_CERT_PRUNE, STEP_CERT_APPLY = range(6)
PACK_CHANGED, PACK_REMOVED = 0, 1


def partition_layout(n: int, world: int, rank: int):
    """(slice, padded, own_lo, own_hi): equal 32-aligned slices of [0, n)."""
    slice_ = ((n + world - 1) // world + 31) // 32 * 32 if n else 0
    lo = min(n, slice_ * rank)
    hi = min(n, slice_ * (rank + 1))
    return slice_, slice_ * world, lo, hi


class _CudaArray:
    """Minimal __cuda_array_interface__ holder for a device buffer we own."""

    def __init__(self, ptr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {
            "shape": (count,), "typestr": typestr, "data": (ptr, False), "version": 3,
            "strides": None,
        }


class DeviceSteps:
    """This rank's share of the solve on its GPU (egs_part_* C-ABI)."""

    def __init__(self, arena: N.GameArena, rank: int, world: int,
                 options: Optional[N.SolverOptions] = None):
        import torch

        options = options or N.SolverOptions()
        opts = options.to_c()
        opts.n_gpus = world
        self.arena = arena
        self.rank, self.world = rank, world
        self._view = arena.view()
        self._part = C.c_void_p()
        lay = N.PartLayout()
        st = N.GpuStats()
        N._check(N.lib.egs_part_create(C.byref(self._view), C.byref(opts), rank, world,
                                       C.byref(self._part), C.byref(lay), C.byref(st)))
        self.upload_seconds = st.upload_seconds
        self.n, self.slice, self.padded = lay.num_vertices, lay.slice, lay.padded
        self.own_lo, self.own_hi = lay.own_lo, lay.own_hi
        self.value_bytes = lay.value_bytes
        typestr = "<i4" if lay.value_bytes == 4 else "<i8"  # bit patterns only
        dev = torch.device("cuda", torch.cuda.current_device())
        count = max(self.padded, 1)
        self.f = torch.as_tensor(_CudaArray(lay.f_dev, count, typestr), device=dev)
        self.stage = torch.as_tensor(_CudaArray(lay.stage_dev, count, typestr), device=dev)
        # sparse exchange: packed (id, value) entries, `entry_words` u64 each
        self.entry_words = max(lay.entry_bytes // 8, 1)
        if world > 1:
            self.send = torch.as_tensor(
                _CudaArray(lay.send_dev, self.slice * self.entry_words + 1, "<i8"), device=dev)
            self.recv = torch.as_tensor(
                _CudaArray(lay.recv_dev, world * self.slice * self.entry_words + 1, "<i8"),
                device=dev)
        self._counts = (C.c_uint64 * 2)()

    def step(self, kind: int, parity: int):
        N._check(N.lib.egs_part_step(self._part, kind, parity, self._counts))
        return int(self._counts[0]), int(self._counts[1])

    def pack(self, which: int, parity: int) -> int:
        cnt = C.c_uint32(0)
        N._check(N.lib.egs_part_pack(self._part, which, parity, C.byref(cnt)))
        return int(cnt.value)

    def unpack(self, counts, stride: int):
        arr = (C.c_uint32 * len(counts))(*counts)
        N._check(N.lib.egs_part_unpack(self._part, arr, stride))

    def reset(self):
        N._check(N.lib.egs_part_reset(self._part))

    def read_measure(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.int64)
        N._check(N.lib.egs_part_read_measure(self._part, out.ctypes.data))
        return out

    def counters(self) -> dict:
        st = N.GpuStats()
        N._check(N.lib.egs_part_counters(self._part, C.byref(st)))
        return st.as_dict()

    def close(self):
        if self._part:
            N.lib.egs_part_destroy(self._part)
            self._part = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TorchComm:
    """All-gather of owned slices and integer all-reduce over torch.distributed.

    ``staged=False``: NCCL, in place on the device tensors.  ``staged=True``:
    any backend (gloo) through host copies -- for tests on CPU or with several
    ranks sharing one GPU."""

    def __init__(self, rank: int, world: int, staged: bool = False, device=None):
        import torch
        import torch.distributed as dist

        self.dist, self.torch = dist, torch
        self.rank, self.world, self.staged = rank, world, staged
        self.device = device
        self.bytes_gathered = 0
        self.collectives = 0

    def allgather(self, t, slice_: int):
        """t[r*slice:(r+1)*slice] of every rank r into t on every rank."""
        self.collectives += 1
        self.bytes_gathered += t.numel() * t.element_size()
        if self.world == 1:
            return
        mine = t.narrow(0, self.rank * slice_, slice_)
        if not self.staged:
            self.dist.all_gather_into_tensor(t, mine)
            # the next step runs on the library's own stream: wait for NCCL
            self.torch.cuda.synchronize(t.device)
            return
        host = mine.detach().to("cpu", copy=True)
        parts = [self.torch.empty_like(host) for _ in range(self.world)]
        self.dist.all_gather(parts, host)
        t.copy_(self.torch.cat(parts).to(t.device))
        self._sync(t)

    def allgather_ints(self, x: int) -> list:
        """Every rank's x (one small collective; its sum is the all-reduce)."""
        self.collectives += 1
        if self.world == 1:
            return [int(x)]
        dev = self.device if (self.device is not None and not self.staged) else "cpu"
        v = self.torch.tensor([int(x)], dtype=self.torch.int64, device=dev)
        out = self.torch.empty(self.world, dtype=self.torch.int64, device=dev)
        self.dist.all_gather_into_tensor(out, v)
        return [int(y) for y in out.tolist()]

    def gather_entries(self, send, recv, n: int):
        """send[:n] of every rank r into recv[r*n:(r+1)*n] on every rank."""
        self.collectives += 1
        self.bytes_gathered += n * self.world * send.element_size()
        if self.world == 1 or n == 0:
            return
        if not self.staged:
            self.dist.all_gather_into_tensor(recv.narrow(0, 0, n * self.world), send.narrow(0, 0, n))
            self.torch.cuda.synchronize(recv.device)
            return
        host = send.narrow(0, 0, n).detach().to("cpu", copy=True)
        parts = [self.torch.empty_like(host) for _ in range(self.world)]
        self.dist.all_gather(parts, host)
        recv.narrow(0, 0, n * self.world).copy_(self.torch.cat(parts).to(recv.device))
        self._sync(recv)

    def _sync(self, t):
        # the library's next step runs on its own non-blocking stream: the
        # copy on torch's stream must have landed
        if t.is_cuda:
            self.torch.cuda.synchronize(t.device)

    def allreduce_sum(self, x: int) -> int:
        self.collectives += 1
        if self.world == 1:
            return int(x)
        dev = self.device if (self.device is not None and not self.staged) else "cpu"
        v = self.torch.tensor([int(x)], dtype=self.torch.int64, device=dev)
        self.dist.all_reduce(v)
        return int(v.item())


@dataclass
class PartitionReport:
    measure: np.ndarray
    rounds: int = 0
    cert_attempts: int = 0
    cert_passes: int = 0
    certified: int = 0
    wall_seconds: float = 0.0
    collectives: int = 0
    bytes_gathered: int = 0
    kernel_launches: int = 0
    sparse_exchanges: int = 0
    counters: dict = field(default_factory=dict)


def solve_partitioned(steps, comm, certify: bool = True, cert_interval: int = 1,
                      cert_growth: int = 4,
                      round_budget: Optional[int] = None,
                      timeout_seconds: float = 0.0) -> PartitionReport:
    """The dense schedule of k_solve (egs_solve.cuh), one step at a time.

    ``steps`` is this rank's share (``DeviceSteps`` in the product);
    ``comm`` exchanges the owned slices (``TorchComm``).  Every rank returns
    the same least progress measure."""
    t0 = time.perf_counter()
    launches = 0
    step_fn = steps.step

    def step(kind, par):
        nonlocal launches
        launches += 1  # one k_part_step launch per call
        return step_fn(kind, par)

    sparse_exchanges = 0

    def exchange(which, parity, counts):
        """Bring every rank's marked values into the replicas: (id, value)
        entries when few changed, else the whole owned slices of f."""
        nonlocal sparse_exchanges
        maxc = max(counts)
        if maxc == 0 or comm.world == 1:
            return
        ew = getattr(steps, "entry_words", 1)
        dense_words = steps.slice * steps.f.element_size() / 8
        if maxc * ew * 2 > dense_words or not hasattr(steps, "pack"):
            comm.allgather(steps.f, steps.slice)
            return
        n = steps.pack(which, parity)
        assert n == counts[comm.rank], "pack count differs from the step's count"
        comm.gather_entries(steps.send, steps.recv, maxc * ew)
        steps.unpack(counts, maxc)
        sparse_exchanges += 1

    parity = 0
    counts = comm.allgather_ints(step(STEP_ROUND1, parity)[0])
    changed = sum(counts)
    rounds = 1
    K = cert_interval if cert_interval > 0 else 1
    next_cert = K
    attempts = passes = certified = 0
    while changed:
        step(STEP_COMMIT, parity)
        exchange(PACK_CHANGED, parity, counts)
        if round_budget is not None and rounds >= round_budget:
            raise N.BoundExhaustedError(
                f"round budget of {round_budget} exhausted before reaching a fixpoint")
        if timeout_seconds and time.perf_counter() - t0 > timeout_seconds:
            raise N.TimeoutError_("solve timed out")
        if certify and rounds >= next_cert:
            attempts += 1
            # candidates carry a mark in f (egs_solve.cuh CandFlag): the passes
            # read the other ranks' marks, so f is exchanged after each step
            step(STEP_CERT_INIT, parity)
            comm.allgather(steps.f, steps.slice)
            while True:
                rc = comm.allgather_ints(step(STEP_CERT_PRUNE, parity)[1])
                removed = sum(rc)
                exchange(PACK_REMOVED, parity, rc)
                passes += 1
                if removed == 0:
                    break
            cert = comm.allreduce_sum(step(STEP_CERT_APPLY, parity)[0])
            comm.allgather(steps.f, steps.slice)
            certified += cert
            K = min(cert_growth * K, 64)  # the geometric schedule of k_solve
            next_cert = rounds + K
        parity ^= 1
        counts = comm.allgather_ints(step(STEP_LIFT, parity)[0])
        changed = sum(counts)
        rounds += 1
    f = steps.read_measure()
    return PartitionReport(
        measure=f, rounds=rounds, cert_attempts=attempts, cert_passes=passes,
        certified=certified, wall_seconds=time.perf_counter() - t0,
        collectives=comm.collectives, bytes_gathered=comm.bytes_gathered,
        sparse_exchanges=sparse_exchanges,
        kernel_launches=launches,
        counters=steps.counters() if hasattr(steps, "counters") else {},
    )
