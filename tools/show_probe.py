"""Pretty-print probe_solve.py JSON lines."""
import json
import sys

for path in sys.argv[1:]:
    print("==", path)
    for line in open(path):
        if not line.startswith("{"):
            print(line.rstrip())
            continue
        d = json.loads(line)
        print(f"{d['config']} {d['mode']:6s} r={d['rounds']:3d} d/s={d['dense_rounds']}/{d['sparse_rounds']} "
              f"cert={d['cert_attempts']}/{d['cert_passes']} ({d['certified']}) "
              f"solve={d['solve_seconds'] * 1e3:8.3f}ms seed={d['seed_seconds'] * 1e3:.3f} "
              f"lift={d['lift_seconds'] * 1e3:.3f} cert={d['cert_seconds'] * 1e3:.3f} "
              f"act={d['activate_seconds'] * 1e3:.3f} GB/s={d['solve_GBps']:.0f} "
              f"liftGB/s={d['lift_GBps']:.0f} grid={d['grid_ctas']} up={d['upload_s']:.3f}")
        if "lift_sub_seconds" in d:
            print("     lift sub (H/M/L0/L1/sparse ms):",
                  " ".join(f"{x * 1e3:.3f}" for x in d["lift_sub_seconds"]))
        if "phase_detail_seconds" in d:
            print("     commit / cert init, dense, sparse, apply (ms):",
                  " ".join(f"{x * 1e3:.3f}" for x in d["phase_detail_seconds"]))
