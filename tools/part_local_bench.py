"""Timing of the partitioned solve with several ranks in ONE process sharing
the visible GPU (distributed.solve_local): a path check of the device-side
exchange on a single-GPU box -- the ranks split one GPU's SMs, so this is not
a scaling number.  usage: python tools/part_local_bench.py [C4] [world]"""
import json
import statistics
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1710_03647_b200 as egs  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_1710_03647_b200.distributed import solve_local  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
kind, args = CONFIGS[cfg]
a = getattr(egs.GameArena, kind)(*args, 1, pinned=True)
with egs.DeviceSolver(a, egs.SolverOptions(device=0)) as ds:
    ds.solve()
    want = ds.read_measure()
    single = statistics.median(ds.solve().solve_seconds for _ in range(5))
t0 = time.perf_counter()
reps, parts = solve_local(a, world, options=egs.SolverOptions(device=0))
create_solve = time.perf_counter() - t0
times = []
for _ in range(5):
    reps, parts = solve_local(a, world, parts=parts)
    times.append(max(r.solve_seconds for r in reps))
ok = all(np.array_equal(r.measure, want) for r in reps)
print(json.dumps({
    "config": cfg, "world": world, "identical_to_single_gpu": ok,
    "single_gpu_ms": single * 1e3, "partitioned_ms_median": statistics.median(times) * 1e3,
    "first_create_and_solve_s": create_solve,
    "rounds": [r.rounds for r in reps], "edges_owned": [r.edges_owned for r in reps],
    "edges_relaxed": [r.edges_relaxed for r in reps], "h2d_bytes": [r.h2d_bytes for r in reps],
    "note": "ranks share ONE GPU (each a half-size persistent grid): exercises the device "
            "exchange, not a multi-GPU scaling measurement"}))
for p in parts:
    p.close()
