"""Full-size golden vectors of the BASELINE configs the reference CPU solver
can finish: C2 = fixed(10^6, 8, W=10^3), C5 = fixed(10^6, 8, W=10^5),
C3 = rmat(22, 16, W=100) and the C4-shape pin F16 = fixed(10^6, 16, W=100).

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
output bytes against them.  C4 itself is out of reach of the reference
(projected days of sweeps); it is pinned by F16 (same
generator, 16x smaller) and by the GPU's certificate-free value iteration
(tests/golden/make_golden_plain.py).
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

# name -> (generator, args); "F16" is the C4-shape pin SURVEY.md §8(d) asks for
# (full CPU parity on the same generator at V = 10^6, d = 16, W = 100).
FULL = {"C2": ("fixed", (1_000_000, 8, 1000)), "C5": ("fixed", (1_000_000, 8, 100_000)),
        "F16": ("fixed", (1_000_000, 16, 100)), "C3": ("rmat", (22, 16, 100))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--timeout", type=float, default=1800.0)
    ap.add_argument("--workers", type=int, default=0, help="0 = every host thread")
    ap.add_argument("configs", nargs="?", default="C2,C5")
    args = ap.parse_args()
    ref = RefLib()
    fnv = Oracle().fnv1a64  # the C FNV-1a-64 of oracle/egs_oracle.c (12 MB texts)
    workers = args.workers or os.cpu_count() or 1
    out = {}
    if os.path.exists(args.out):  # resume: keep the configs already finished
        with open(args.out) as fh:
            out = json.load(fh)
    for cfg in args.configs.split(","):
        gen, gargs = FULL[cfg]
        key = f"{gen}/" + "/".join(map(str, gargs)) + "/1"
        if key in out:
            continue
        a = getattr(ref, gen)(*gargs, 1)
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
