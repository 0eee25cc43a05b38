"""A/B timing of library builds (dev tool): for each EGS_LIB path, the median
device-resident solve time and per-phase split of the given configs.
    python tools/ab_time.py C4,C3 default scratch_libs/x/libegs_b200.so ..."""
import json
import os
import statistics
import subprocess
import sys

CHILD = r'''
import sys, json, statistics
sys.path.insert(0, ".")
import paper_1710_03647_b200 as egs
from bench import CONFIGS
for cfg in sys.argv[1].split(","):
    kind, args = CONFIGS[cfg]
    a = getattr(egs.GameArena, kind)(*args, 1, pinned=True)
    with egs.DeviceSolver(a, egs.SolverOptions(device=0)) as ds:
        for _ in range(3): ds.solve()
        st = [ds.solve() for _ in range(int(sys.argv[2]))]
        f = ds.read_measure()
        ok = ds.is_fixpoint(f) and ds.is_progress_measure(f)
    ms = statistics.median(s.solve_seconds for s in st) * 1e3
    d = st[-1].as_dict()
    print(json.dumps({"cfg": cfg, "ms": round(ms, 4), "min_ms": round(min(s.solve_seconds for s in st) * 1e3, 4),
                      "ok": ok, "rounds": d["rounds"], "cert_edges": d.get("cert_edges"),
                      "phases_us": [round(x * 1e6, 1) for x in d.get("phase_detail_seconds", [])],
                      "tops": int((f == (1 << 63) - 1).sum())}), flush=True)
'''

def main():
    cfgs = sys.argv[1]
    steps = os.environ.get("AB_STEPS", "30")
    for rep in range(int(os.environ.get("AB_REPS", "2"))):
        for lib in sys.argv[2:]:
            env = dict(os.environ)
            if lib != "default":
                env["EGS_LIB"] = os.path.abspath(lib)
            out = subprocess.run([sys.executable, "-c", CHILD, cfgs, steps], env=env,
                                 capture_output=True, text=True, timeout=600)
            for line in out.stdout.splitlines():
                print(json.dumps({"lib": lib, "rep": rep, **json.loads(line)}), flush=True)
            if out.returncode:
                print(lib, "FAILED", out.stderr[-2000:], flush=True)

if __name__ == "__main__":
    main()
