"""Minimal ncu target: one device-resident solve of a canonical config
(default C4).  Usage: python tools/ncu_target.py [C4] [solves] [round_budget]
A round budget stops the kernel after that many rounds (e.g. 1: round 1 and
its commit only), so a capture isolates the early phases."""
import sys

sys.path.insert(0, ".")
import paper_1710_03647_b200 as egs  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
kind, args = CONFIGS[cfg]
a = getattr(egs.GameArena, kind)(*args, 1, pinned=True)
budget = int(sys.argv[3]) if len(sys.argv) > 3 else 0
opts = egs.SolverOptions(sweep_bound=budget) if budget else None
with egs.DeviceSolver(a, opts) as ds:
    for _ in range(reps):
        try:
            st = ds.solve()
            print(cfg, st.as_dict())
        except egs.BoundExhaustedError:
            print(cfg, "stopped at the round budget")
