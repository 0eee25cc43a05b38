"""Full-size golden vectors of the BASELINE configs the reference CPU solver
can finish: C2 = fixed(10^6, 8, W=10^3) and C5 = fixed(10^6, 8, W=10^5).

The COMPILED REFERENCE (oracle/_ref/libegsolve_ref.so, built from
/root/reference/proj/src by the Makefile) runs solve_sweep on every host
thread to its fixpoint (~2.3e5 sweeps, ~15 min each on the GPU box's 16
threads, which is why this runs there, under gpurun: the .so travels with the
snapshot).  It records what the reference prints -- the write_solution text's
length, FNV-1a-64 and SHA-256, the number of top vertices, the sum and max of
finite credits -- plus the reference's own sweep count and wall time.

    python tests/golden/make_golden_full.py --out gpurun_out/golden_full.json [C2,C5]

Merge the output into tests/golden/golden.json (keys fixed/<n>/<d>/<W>/1);
tests/test_gpu_parity.py::test_full_size_golden checks the GPU solver's
output bytes against them.  C3 and C4 are out of reach of the reference
(projected days of sweeps).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_bindings import INT64_MAX, Oracle, RefLib  # noqa: E402

FULL = {"C2": (1_000_000, 8, 1000), "C5": (1_000_000, 8, 100_000)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--timeout", type=float, default=1800.0)
    ap.add_argument("configs", nargs="?", default="C2,C5")
    args = ap.parse_args()
    ref = RefLib()
    fnv = Oracle().fnv1a64  # the C FNV-1a-64 of oracle/egs_oracle.c (12 MB texts)
    workers = os.cpu_count() or 1
    out = {}
    for cfg in args.configs.split(","):
        n, d, W = FULL[cfg]
        key = f"fixed/{n}/{d}/{W}/1"
        a = ref.fixed(n, d, W, 1)
        t0 = time.time()
        f, st, wall = ref.solve(a, RefLib.SWEEP, workers=workers, timeout=args.timeout)
        sol = ref.write_solution(a, f).encode()
        fin = f[f != INT64_MAX]
        out[key] = {
            "n": a.n, "m": a.m, "credit_cap": ref.credit_cap(a),
            "solution_bytes": len(sol), "solution_fnv": f"{fnv(sol):016x}",
            "solution_sha256": hashlib.sha256(sol).hexdigest(),
            "tops": int((f == INT64_MAX).sum()), "sum_finite": int(fin.sum()),
            "max_finite": int(fin.max()) if fin.size else 0,
            "ref_solver": f"solve_sweep workers={workers}", "ref_rounds": st["rounds"],
            "ref_wall_s": round(wall, 3), "config": cfg,
        }
        print(key, json.dumps(out[key]), f"{time.time() - t0:.1f}s", flush=True)
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
