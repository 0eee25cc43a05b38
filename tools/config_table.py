"""Per-config table of the five BASELINE.json configs on one B200, the compiled
reference beside each (run under gpurun from the repo root):

    python tools/config_table.py [--out gpurun_out/configs.jsonl]

For every config: the device-resident time-to-fixpoint (median of K solves,
CUDA events) and GTEPS, the one-shot e2e time through egs_gpu_solve (pinned
host arena), the fixpoint / progress-measure checks of the result on the
device (egs_ctx_is_fixpoint, the EPM verifier of measure_ops.cpp:33-41), and
the reference solve_sweep on all host threads: to its fixpoint where it
finishes (C1: median of 5, plus byte parity of write_solution), else a
bounded sample of sweeps (s/sweep, edge-relax rate) and, where SURVEY.md §0.4
gives a sweep count, the projected time to fixpoint.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for _p in (ROOT, os.path.join(ROOT, "tests")):
    if _p not in sys.path:
        sys.path.insert(0, _p)

from bench import CONFIGS, workload_name  # noqa: E402

# reference sweeps to the fixpoint: C2 / C5 measured (the reference run to its
# fixpoint on the GPU box host, tests/golden/make_golden_full.py, 16 threads),
# C3 measured (the same on the build container, 4 threads:
# profiles/r02_golden_full_f16_c3.txt); C4 from the SURVEY.md §0.4
# regression (the GPU's own in-place sweep of the same iteration took
# 1,914,825 rounds, profiles/r02_golden_plain_gpu_c4_sweep.json)
PROJECTED_SWEEPS = {"C2": 228296, "C3": 22036, "C4": 2.1e6, "C5": 224879}
SWEEP_SOURCE = {"C2": "measured (reference to its fixpoint)",
                "C3": "measured (reference to its fixpoint, 4 threads)",
                "C5": "measured (reference to its fixpoint)",
                "C4": "SURVEY.md §0.4 regression"}
SAMPLE_SWEEPS = {"C2": 50, "C3": 5, "C4": 3, "C5": 50}


def log(s):
    print(s, file=sys.stderr, flush=True)


def ours(cfg, steps):
    import numpy as np
    import paper_1710_03647_b200 as egs
    kind, args = CONFIGS[cfg]
    arena = getattr(egs.GameArena, kind)(*args, 1, pinned=True)
    opts = egs.SolverOptions(device=0)
    with egs.DeviceSolver(arena, opts) as ds:
        for _ in range(3):
            ds.solve()
        st = [ds.solve() for _ in range(steps)]
        f = ds.read_measure()
        fix = ds.is_fixpoint(f)
        epm = ds.is_progress_measure(f)
        text = ds.write_solution()
    ms = statistics.median(s.solve_seconds for s in st) * 1e3
    last = st[-1]
    out, _owner = egs.pinned_empty(arena.num_vertices)  # keep the owner alive
    egs.solve(arena, options=opts, out=out)
    e2e = []
    for _ in range(5):
        t0 = time.perf_counter()
        egs.solve(arena, options=opts, out=out)
        e2e.append(time.perf_counter() - t0)
    assert np.array_equal(out, f)
    host_text = egs.write_solution(arena, f)
    top = int((f == np.iinfo(np.int64).max).sum())
    fin = f[f != np.iinfo(np.int64).max]
    return {
        "vertices": arena.num_vertices, "edges": arena.num_edges,
        "time_to_fixpoint_ms": ms, "gteps": last.edges_relaxed / (ms * 1e-3) / 1e9,
        "rounds": last.rounds, "dense_rounds": last.dense_rounds,
        "sparse_rounds": last.sparse_rounds, "certified": last.certified,
        "edges_relaxed": last.edges_relaxed, "value_bits": last.value_bits,
        "e2e_ms_median": statistics.median(e2e) * 1e3,
        "fixpoint": fix, "progress_measure": epm,
        "device_text_equals_host_text": text == host_text,
        "top": top, "finite_sum": int(fin.sum()), "finite_max": int(fin.max()) if fin.size else 0,
    }, f, host_text


def reference(cfg, f_gpu, text_gpu):
    from oracle_bindings import RefLib
    ref = RefLib()
    kind, args = CONFIGS[cfg]
    a = getattr(ref, kind)(*args, 1)
    workers = os.cpu_count() or 1
    r = {"cores": workers, "kind": "reference solve_sweep"}
    if cfg == "C1":
        walls, rounds = [], None
        for _ in range(5):
            f, st, wall = ref.solve(a, variant=RefLib.SWEEP, workers=workers)
            walls.append(wall)
            rounds = st["rounds"]
        import numpy as np
        r.update(time_to_fixpoint_s=statistics.median(walls), sweeps=rounds,
                 measure_bit_exact=bool(np.array_equal(f, f_gpu)),
                 solution_bytes_identical=ref.write_solution(a, f) == text_gpu,
                 edge_relax_per_s=rounds * a.m / statistics.median(walls))
        return r
    k = SAMPLE_SWEEPS[cfg]
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        try:
            ref.solve(a, variant=RefLib.SWEEP, workers=workers, sweep_bound=k)
        except RuntimeError as e:
            if getattr(e, "code", None) != 5:
                raise
        times.append(time.perf_counter() - t0)
    sps = statistics.median(times[1:]) / k
    r.update(sample=f"{k} sweeps x 2 timed (after 1 warm-up)", s_per_sweep=sps,
             edge_relax_per_s=a.m / sps,
             progress_measure_of_gpu_result=ref.is_progress_measure(a, f_gpu))
    if cfg in PROJECTED_SWEEPS:
        r["time_to_fixpoint_s_projected"] = sps * PROJECTED_SWEEPS[cfg]
        r["projection"] = (f"s/sweep x {PROJECTED_SWEEPS[cfg]:.7g} sweeps "
                           f"({SWEEP_SOURCE[cfg]})")
    return r


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out", default=None)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--configs", default="C1,C2,C3,C4,C5")
    a = p.parse_args()
    lines = []
    for cfg in a.configs.split(","):
        t0 = time.perf_counter()
        o, f, text = ours(cfg, a.steps)
        log(f"{cfg}: ours {o['time_to_fixpoint_ms']:.3f} ms ({time.perf_counter() - t0:.1f} s)")
        rr = reference(cfg, f, text)
        line = {"config": cfg, "workload": workload_name(cfg), "ours": o, "reference": rr}
        ttf = rr.get("time_to_fixpoint_s") or rr.get("time_to_fixpoint_s_projected")
        if ttf:
            line["time_to_fixpoint_speedup"] = {
                "device_resident": ttf / (o["time_to_fixpoint_ms"] * 1e-3),
                "e2e": ttf / (o["e2e_ms_median"] * 1e-3),
                "reference_measured": "time_to_fixpoint_s" in rr}
        print(json.dumps(line), flush=True)
        lines.append(line)
    if a.out:
        with open(a.out, "w") as fh:
            for ln in lines:
                fh.write(json.dumps(ln) + "\n")


if __name__ == "__main__":
    main()
