"""Benchmark of the energy-game solve path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C4] [--no-cpu-baseline]

A step is one solve of the initial-credit problem to its least fixpoint
(seed -> lift rounds -> fixpoint) over one synthetic arena.
The workload is C4 = fixed(1.6e7 vertices, out-degree 16, W=100, seed 1), the
16M-vertex game BASELINE.json's target is quoted on; the
other configs are parity cases (tests/), not bench lines.

Our arm prints ONE JSON line on rank 0:
  value      GTEPS = edges relaxed inside lifts / device time-to-fixpoint,
             arena resident in HBM (CUDA events on the solver's stream).
  e2e        the same metric through the C-ABI one-shot call egs_gpu_solve
             with pinned HOST buffers: arena H2D, device CSC build, solve and
             the D2H of the int64 measure all inside the timed region.
  roofline   the lift kernels (dominant): algorithmic bytes (SURVEY.md §8d,
             DESIGN.md §4) / their CUDA-event time, against measured HBM peak.
  cpu_baseline  the compiled reference (oracle/_ref, solve_sweep on all host
             threads) on a bounded sample of the same arena: S sweeps.
`--impl reference` times only that reference CPU path, same metric and unit.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
for _p in (ROOT, os.path.join(ROOT, "tests")):
    if _p not in sys.path:
        sys.path.insert(0, _p)

METRIC = "time-to-fixpoint (s) and GTEPS edges-relaxed/sec at 1/2/4/8 B200 vs CPU ref"
UNIT = "GTEPS"
CONFIGS = {
    "C1": ("fixed", (10_000, 4, 100)),
    "C2": ("fixed", (1_000_000, 8, 1000)),
    "C3": ("rmat", (22, 16, 100)),
    "C4": ("fixed", (16_000_000, 16, 100)),
    "C5": ("fixed", (1_000_000, 8, 100_000)),
}
# Survey projection of reference sweeps-to-fixpoint on C4;
# the GPU's in-place sweep (the reference's iteration, certify=False, mode
# sweep) reached the fixpoint in 1,914,825 rounds
# (profiles/r02_golden_plain_gpu_c4_sweep.json).
C4_PROJECTED_REF_SWEEPS = 2.1e6
FALLBACK_HBM_GBS = 6650.0


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def workload_name(cfg):
    kind, args = CONFIGS[cfg]
    if kind == "fixed":
        n, d, W = args
        return f"{cfg} fixed(n={n}, d={d}, W={W}, seed=1)"
    s, ef, W = args
    return f"{cfg} rmat(scale={s}, ef={ef}, W={W}, seed=1)"


# ----------------------------------------------------------- clocks ----
class ClockSampler:
    """NVML SM clock + throttle reasons sampled every 5 ms while running."""

    REASONS = {
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
    }

    def __init__(self, index=0):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.nv is not None:
            self._stop.clear()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(self.reasons),
            "samples": len(self.samples),
        }


# ----------------------------------------------------- distributed ----
def dist_setup(n_gpus, backend):
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            import torch
            ndev = max(1, torch.cuda.device_count())
            torch.cuda.set_device(env_int("LOCAL_RANK", 0) % ndev)
            if ndev < env_int("LOCAL_WORLD_SIZE", world):
                # ranks sharing a GPU (a functional run on a smaller box):
                # NCCL refuses duplicate devices; the plumbing is gloo's
                backend = "gloo"
        dist.init_process_group(backend=backend)
    return rank, world


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world, device=None):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    if dist.get_backend() != "nccl":
        device = None  # (gloo reduces host tensors)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, world, device=None):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    if dist.get_backend() != "nccl":
        device = None  # (gloo reduces host tensors)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ------------------------------------------------- reference (CPU) ----
def reference_sample(cfg, sweeps, steps, warmup, log):
    """The unmodified reference solve_sweep (oracle/_ref) on all host threads,
    each step bounded to `sweeps` sweeps (BoundExhaustedError ends it)."""
    from oracle_bindings import RefLib
    ref = RefLib()
    kind, args = CONFIGS[cfg]
    t0 = time.perf_counter()
    a = getattr(ref, kind)(*args, 1)
    log(f"reference arena built in {time.perf_counter() - t0:.1f} s")
    workers = os.cpu_count() or 1
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        try:
            ref.solve(a, variant=RefLib.SWEEP, workers=workers, sweep_bound=sweeps)
            done = True
        except RuntimeError as e:
            if getattr(e, "code", None) != 5:
                raise
            done = False
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
        log(f"reference step {i}: {dt:.3f} s ({'fixpoint' if done else f'{sweeps} sweeps'})")
    m = a.m
    total = sum(times)
    gteps = sweeps * m * len(times) / total / 1e9
    return {
        "value": gteps,
        "unit": UNIT,
        "cores": workers,
        "kind": "reference",
        "s_per_sweep": total / len(times) / sweeps,
        "sample": f"{sweeps} sweeps of reference solve_sweep (workers={workers}) on "
                  f"{workload_name(cfg)}, {len(times)} timed samples; edges relaxed = sweeps x |E|",
        "time_to_fixpoint_s_projected": (total / len(times) / sweeps * C4_PROJECTED_REF_SWEEPS
                                         if cfg == "C4" else None),
    }


def run_reference_arm(a):
    rank, world = dist_setup(a.gpus, "gloo")
    if rank != 0:
        return
    log = (lambda s: print(s, file=sys.stderr, flush=True))
    cb = reference_sample(a.config, a.ref_sweeps, a.steps, a.warmup, log)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": cb["s_per_sweep"] * a.ref_sweeps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int64", "data": "synthetic",
        "config": {"workload": workload_name(a.config), "sample_sweeps": a.ref_sweeps},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "time_to_fixpoint_s_projected": cb["time_to_fixpoint_s_projected"],
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------- our arm ----
def h2d_bytes(arena):
    """Bytes that cross PCIe per upload: offsets (u64) + owners + targets (u32)
    + weights narrowed on the host to int8/int16/int32 by max |w|
    (egs_solver.cu upload_weights)."""
    n, m, mw = arena.num_vertices, arena.num_edges, arena.max_abs_weight
    wb = 1 if mw <= 127 else 2 if mw <= 32767 else 4
    return (n + 1) * 8 + n + m * 4 + m * wb

def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        for k in ("hbm_gbs", "hbm_GBs", "hbm_copy_gbs"):
            if k in d:
                return float(d[k]), "measured"
    except Exception:
        pass
    return FALLBACK_HBM_GBS, "fallback"


def source_digest():
    """SHA-256 over the library's sources and build recipe (csrc/, the C-ABI
    header, Makefile): what determines k_solve's code, unlike the .so's own
    hash, which also changes with the build directory (-lineinfo paths)."""
    import glob
    import hashlib
    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(ROOT, "paper_1710_03647_b200", "csrc", "*"))) + [
        os.path.join(ROOT, "include", "egs_gpu.h"), os.path.join(ROOT, "Makefile")]
    for f in files:
        if f.endswith((".cu", ".cuh", ".cpp", ".h")) or f.endswith("Makefile"):
            h.update(os.path.relpath(f, ROOT).encode())
            with open(f, "rb") as fh:
                h.update(fh.read())
    return h.hexdigest()


def load_traffic():
    """Per-launch DRAM bytes of k_solve from the committed ncu capture
    (tools/summarize_profile.py), used only when it was captured from the
    very sources this run's library is built from (source digest stamp);
    otherwise None."""
    p = os.path.join(ROOT, "profiles", "lift_traffic.json")
    try:
        with open(p) as fh:
            t = json.load(fh)
    except Exception:
        return None, "no committed ncu capture"
    if t.get("source_digest") != source_digest():
        return None, "committed ncu capture is of other library sources"
    return t, t.get("source")


def run_our_arm(a):
    import numpy as np
    import torch

    import paper_1710_03647_b200 as egs

    rank, world = dist_setup(a.gpus, "nccl")
    dev = env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(dev)
    log = (lambda s: print(f"[rank {rank}] {s}", file=sys.stderr, flush=True))
    kind, args = CONFIGS[a.config]
    t0 = time.perf_counter()
    arena = getattr(egs.GameArena, kind)(*args, 1, pinned=True)
    n, m = arena.num_vertices, arena.num_edges
    log(f"generated {workload_name(a.config)}: n={n} m={m} in {time.perf_counter() - t0:.1f} s")
    opts = egs.SolverOptions(device=dev)

    # ---- device-resident solves: value --------------------------------
    ds = egs.DeviceSolver(arena, opts)
    for _ in range(a.warmup):
        ds.solve()
    barrier(world)
    torch.cuda.synchronize()
    stats = []
    with ClockSampler(dev) as clk:
        for _ in range(a.steps):
            stats.append(ds.solve())
        torch.cuda.synchronize()
    barrier(world)
    dev_s = sum(s.solve_seconds for s in stats)
    dev_s = max_over_ranks(dev_s, world, "cuda")
    edges = sum(s.edges_relaxed for s in stats)
    edges_all = sum_over_ranks(edges, world, "cuda")
    value = edges_all / dev_s / 1e9
    launches = sum(s.kernel_launches for s in stats)
    algo_bytes = sum(s.algo_bytes for s in stats)
    algo_s8d = sum(s.algo_bytes_s8d for s in stats)
    lift_bytes = sum(s.lift_bytes for s in stats)
    lift_s = sum(s.lift_seconds for s in stats)
    cert_s = sum(s.cert_seconds for s in stats)
    act_s = sum(s.activate_seconds for s in stats)
    seed_s = sum(s.seed_seconds for s in stats)
    last = stats[-1]
    f_dev = ds.read_measure()
    ds.close()

    # ---- end to end through the C-ABI one-shot call: e2e ---------------
    out, _owner = egs.pinned_empty(n)
    h2d = h2d_bytes(arena)
    # the measure crosses PCIe as the device's values (4 bytes each when they
    # are 32-bit) and is widened to int64 on the host (egs_solver.cu ctx_read)
    d2h = n * (4 if last.value_bits == 32 else 8)
    for _ in range(max(2, a.warmup)):
        egs.solve(arena, options=opts, out=out)
    barrier(world)
    e2e_t, e2e_edges = 0.0, 0
    e2e_steps = []
    with clk:  # the same sampler: clocks under load in both timed regions
        for _ in range(a.e2e_steps):
            t1 = time.perf_counter()
            rep = egs.solve(arena, options=opts, out=out)
            e2e_steps.append(time.perf_counter() - t1)
            e2e_edges += rep.gpu["edges_relaxed"]
    e2e_t = sum(e2e_steps)
    log("e2e steps (ms): " + " ".join(f"{x * 1e3:.1f}" for x in e2e_steps))
    barrier(world)
    e2e_t = max_over_ranks(e2e_t, world, "cuda")
    e2e_edges = sum_over_ranks(e2e_edges, world, "cuda")
    assert np.array_equal(out, f_dev), "one-shot and resident solves disagree"

    peak, peak_kind = load_peaks()
    # The whole solve is one persistent launch of k_solve.  `achieved` is
    # SURVEY.md §8(d)'s algorithmic bytes exactly (edges relaxed x (8 + s) +
    # applications x (4 + 2s) + activations x 4) over the launch's
    # CUDA-event duration; `extended` adds the certificate's and round 1's
    # bytes; `dram` is the measured DRAM traffic of the same
    # build (ncu, stamped with the library's SHA-256) over the same time.
    nl = max(launches, 1)
    achieved = algo_s8d / dev_s / 1e9 if dev_s > 0 else 0.0
    ext_gbs = algo_bytes / dev_s / 1e9 if dev_s > 0 else 0.0
    lift_gbs = lift_bytes / lift_s / 1e9 if lift_s > 0 else 0.0
    traffic, traffic_src = load_traffic()
    tb = (traffic or {}).get("bytes_per_launch")
    dram_gbs = tb / (dev_s / nl) / 1e9 if tb and dev_s > 0 else None
    roofline = {
        "kernel": "k_solve (persistent solve kernel, DESIGN.md §4)",
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "peak_source": f"{peak_kind} HBM copy bandwidth",
        "traffic": tb,
        "traffic_source": traffic_src,
        "algorithmic_bytes_per_launch": algo_s8d / nl,
        "avg_launch_ms": dev_s / nl * 1e3,
        "frac_algorithmic_s8d": achieved / peak,
        "frac_dram": dram_gbs / peak if dram_gbs else None,
        "extended": {"achieved": ext_gbs, "frac": ext_gbs / peak,
                     "bytes_per_launch": algo_bytes / nl,
                     "what": "§8(d) figures plus round 1 and certificate bytes (DESIGN.md §4)"},
        "lift_phases": {"achieved": lift_gbs, "frac": lift_gbs / peak,
                        "bytes_per_launch": lift_bytes / nl,
                        "ms_per_launch": lift_s / nl * 1e3,
                        "what": "lift phases only, edge records at their stored size"},
    }

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": dev_s / a.steps * 1e3,
        "time_to_fixpoint_s": dev_s / a.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32" if last.value_bits == 32 else "u64",
        "data": "synthetic (canonical splitmix64 generator, SURVEY.md Appendix B)",
        "config": {
            "workload": workload_name(a.config), "vertices": n, "edges": m,
            "value_bits": last.value_bits, "grid_ctas": last.grid_ctas,
            "parallelism": "replicas" if world > 1 else "single-gpu",
            "l2": "inputs larger than L2 (edge records 8 B x |E| >> 126 MB); no flush",
        },
        "solve": {
            "rounds": last.rounds, "dense_rounds": last.dense_rounds,
            "sparse_rounds": last.sparse_rounds, "edges_relaxed": last.edges_relaxed,
            "witness_checks": last.witness_checks, "certified": last.certified,
            "cert_passes": last.cert_passes, "seed_ms": seed_s / a.steps * 1e3,
            "lift_ms": lift_s / a.steps * 1e3,
            "cert_ms": cert_s / a.steps * 1e3, "activate_ms": act_s / a.steps * 1e3,
        },
        "e2e": {"value": e2e_edges / e2e_t / 1e9, "unit": UNIT,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_t / a.e2e_steps * 1e3,
                "api": "egs_gpu_solve (include/egs_gpu.h), pinned host arena"},
        "gpu_launches": launches,
        "roofline": roofline,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        del arena
        cb = reference_sample(a.config, a.ref_sweeps, a.cpu_steps, 1, log)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        if cb["time_to_fixpoint_s_projected"]:
            line["cpu_baseline"]["time_to_fixpoint_s_projected"] = cb["time_to_fixpoint_s_projected"]
            line["cpu_baseline"]["projection"] = (
                f"s/sweep x {C4_PROJECTED_REF_SWEEPS:.2g} sweeps (SURVEY.md §0.4 regression)")
            # the north-star target is a time-to-fixpoint speed-up; GTEPS (the
            # `value`) counts edges relaxed, and the certificate makes the GPU
            # solve relax ~|E| edges where the reference sweeps ~2e6 |E|
            proj = cb["time_to_fixpoint_s_projected"]
            line["time_to_fixpoint_speedup"] = {
                "device_resident": proj / line["time_to_fixpoint_s"],
                "e2e": proj / (line["e2e"]["ms_per_step"] * 1e-3),
                "vs": "reference solve_sweep on all host cores, projected (cpu_baseline)",
            }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_our_arm_partitioned(a):
    """N > 1 (torchrun, one process per GPU): the partitioned solve of the same
    C4 arena (distributed.py) -- each rank uploads the arena,
    keeps its class-balanced share of the rows, and the ranks exchange raised
    values by NVLink peer stores inside one persistent kernel per rank; the
    host only swaps IPC handles (torch.distributed) and waits.  Strong
    scaling: the total work is the one C4 solve."""
    import numpy as np
    import torch

    import paper_1710_03647_b200 as egs
    from paper_1710_03647_b200.distributed import Partition, TorchComm, solve_distributed

    rank, world = dist_setup(a.gpus, "nccl")
    dev = env_int("LOCAL_RANK", 0) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    log = (lambda s: print(f"[rank {rank}] {s}", file=sys.stderr, flush=True))
    kind, args = CONFIGS[a.config]
    arena = getattr(egs.GameArena, kind)(*args, 1, pinned=True)
    n, m = arena.num_vertices, arena.num_edges
    opts = egs.SolverOptions(device=dev, workers=world)
    comm = TorchComm()
    red_dev = f"cuda:{dev}"

    part = Partition(arena, rank, world, opts)
    part.connect(comm.allgather_bytes(part.export()))
    barrier(world)
    log(f"plan: rank_lo={part.plan['rank_lo']} edges={part.plan['edges']}")
    for _ in range(a.warmup):
        rep = solve_distributed(arena, comm=comm, part=part)
    f_dev = rep.measure
    total_s, edges = 0.0, 0
    with ClockSampler(dev) as clk:
        for _ in range(a.steps):
            barrier(world)
            rep = solve_distributed(arena, comm=comm, part=part)
            total_s += rep.solve_seconds
            edges += rep.edges_relaxed
    total_s = max_over_ranks(total_s, world, red_dev)
    edges_all = sum_over_ranks(edges, world, red_dev)
    rounds = rep.rounds
    part.close()

    # e2e: this rank's upload (its own rows) + device build, handle exchange,
    # solve, D2H
    h2d_rank = 0
    e2e_t, e2e_edges = 0.0, 0
    for _ in range(a.e2e_steps):
        barrier(world)
        t1 = time.perf_counter()
        r = solve_distributed(arena, opts, comm=comm)
        e2e_t += time.perf_counter() - t1
        e2e_edges += r.edges_relaxed
        h2d_rank = r.h2d_bytes
        assert np.array_equal(r.measure, f_dev)
    e2e_t = max_over_ranks(e2e_t, world, red_dev)
    e2e_edges = sum_over_ranks(e2e_edges, world, red_dev)
    line = {
        "metric": METRIC, "value": edges_all / total_s / 1e9, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": total_s / a.steps * 1e3,
        "time_to_fixpoint_s": total_s / a.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "u32" if arena.credit_cap < 2 ** 31 - 1 else "u64",
        "data": "synthetic (canonical splitmix64 generator, SURVEY.md Appendix B)",
        "config": {"workload": workload_name(a.config), "vertices": n, "edges": m,
                   "parallelism": f"class-balanced vertex partition x{world}, "
                                  "device-side exchange (NVLink peer stores, cross-rank "
                                  "barriers in peer memory)",
                   "l2": "inputs larger than L2; no flush"},
        "solve": {"rounds": rounds, "plan_edges": rep.plan["edges"]},
        "e2e": {"value": e2e_edges / e2e_t / 1e9, "unit": UNIT,
                "h2d_bytes_per_step": int(sum_over_ranks(h2d_rank, world, red_dev)),
                "d2h_bytes_per_step": n * (4 if r.stats.get("value_bits") == 32 else 8) * world,
                "ms_per_step": e2e_t / a.e2e_steps * 1e3,
                "api": "egs_part_create / egs_part_connect / egs_part_solve (include/egs_gpu.h)"},
        "gpu_launches": a.steps,
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    import torch.distributed as dist
    dist.destroy_process_group()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--ref-sweeps", type=int, default=3,
                   help="reference sweeps per timed sample")
    p.add_argument("--cpu-steps", type=int, default=2)
    p.add_argument("--no-cpu-baseline", action="store_true")
    a = p.parse_args()
    if a.warmup < 3:
        p.error("--warmup must be >= 3")
    if a.impl == "reference":
        run_reference_arm(a)
    elif env_int("WORLD_SIZE", 1) > 1:
        run_our_arm_partitioned(a)
    else:
        run_our_arm(a)


if __name__ == "__main__":
    main()
