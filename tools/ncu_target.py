"""Minimal ncu target: one device-resident solve of a canonical config
(default C4).  Usage: python tools/ncu_target.py [C4] [solves]"""
import sys

sys.path.insert(0, ".")
import paper_1710_03647_b200 as egs  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
kind, args = CONFIGS[cfg]
a = getattr(egs.GameArena, kind)(*args, 1, pinned=True)
with egs.DeviceSolver(a) as ds:
    for _ in range(reps):
        st = ds.solve()
    print(cfg, st.as_dict())
