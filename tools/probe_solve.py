"""Quick device probe: solve the canonical configs and print stats (dev tool)."""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import paper_1710_03647_b200 as egs  # noqa: E402

CONFIGS = {
    "C1": ("fixed", (10000, 4, 100)),
    "C2": ("fixed", (1000000, 8, 1000)),
    "C3": ("rmat", (22, 16, 100)),
    "C4": ("fixed", (16000000, 16, 100)),
    "C5": ("fixed", (1000000, 8, 100000)),
}


def main():
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C1", "C2", "C5"]
    modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["auto"]
    for name in names:
        kind, args = CONFIGS[name]
        t0 = time.time()
        a = getattr(egs.GameArena, kind)(*args, 1, pinned=True)
        tg = time.time() - t0
        for mode in modes:
            for certify in (True,):
                kw = json.loads(os.environ.get("EGS_PROBE_OPTS", "{}"))
                ds = egs.DeviceSolver(a, egs.SolverOptions(mode=mode, certify=certify, **kw))
                for rep in range(3):
                    st = ds.solve()
                d = st.as_dict()
                f = ds.read_measure()
                tops = int((f == egs._native.INT64_MAX).sum())
                ds.close()
                d.update(config=name, mode=mode, certify=certify, gen_s=round(tg, 2),
                         upload_s=ds.upload_stats.upload_seconds, tops=tops,
                         lift_GBps=d["lift_bytes"] / max(d["lift_seconds"], 1e-12) / 1e9,
                         solve_GBps=d["algo_bytes"] / max(d["solve_seconds"], 1e-12) / 1e9)
                print(json.dumps(d), flush=True)


if __name__ == "__main__":
    main()
