"""Generate tests/golden/golden.json from the COMPILED REFERENCE (oracle/_ref).

Run where /root/reference exists (after `make`):

    python tests/golden/make_golden.py [--big]

For every instance it records what the reference itself prints:
write_arena / write_solution text length and FNV-1a-64, the number of top
vertices, sum and max of finite credits and credit_cap.  Small fixtures keep
the full solution text.  The GPU box has no /root/reference, so the GPU parity
tests read these committed numbers.  `--big` adds the 10^5-vertex shapes of
SURVEY.md Appendix B (minutes of CPU with the reference sweep solver).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_bindings import INT64_MAX, RefLib, fnv1a64  # noqa: E402

# SPEC.md fixtures as (n, edges, owners).
SPEC_FIXTURES = {
    "G1": (2, [(0, 1, -1), (1, 0, 1)], [0, 1]),
    "p0_selfloop_neg": (1, [(0, 0, -1)], [0]),
    "selfloop_zero": (1, [(0, 0, 0)], [0]),
    "p0_loops_pm1": (1, [(0, 0, -1), (0, 0, 1)], [0]),
    "p1_loops_pm1": (1, [(0, 0, -1), (0, 0, 1)], [1]),
    "strategy_example": (3, [(0, 1, -5), (0, 2, 0), (1, 1, 0), (2, 2, 0)], [0, 0, 0]),
}

SMALL = [
    ("fixed", 10000, 4, 100),      # C1
    ("fixed", 1000, 8, 1000),
    ("fixed", 1000, 8, 100000),
    ("fixed", 2000, 16, 100),
    ("fixed", 3000, 2, 50),
    ("rmat", 12, 16, 100),
    ("rmat", 14, 16, 100),
]
BIG = [
    ("fixed", 100000, 4, 100),
    ("fixed", 100000, 8, 1000),     # C2 shape
    ("fixed", 100000, 16, 100),     # C4 shape
    ("fixed", 100000, 8, 100000),   # C5 shape
    ("rmat", 16, 16, 100),          # C3 shape
]


def summarize(ref: RefLib, a, f, workers: int, rounds: int, wall: float, keep_text: bool):
    sol = ref.write_solution(a, f).encode()
    arena_txt = ref.write_arena(a).encode()
    fin = f[f != INT64_MAX]
    rec = {
        "n": a.n, "m": a.m, "credit_cap": ref.credit_cap(a),
        "arena_bytes": len(arena_txt), "arena_fnv": f"{fnv1a64(arena_txt):016x}",
        "solution_bytes": len(sol), "solution_fnv": f"{fnv1a64(sol):016x}",
        "tops": int((f == INT64_MAX).sum()), "sum_finite": int(fin.sum()),
        "max_finite": int(fin.max()) if fin.size else 0,
        "ref_solver": f"solve_sweep workers={workers}", "ref_rounds": rounds,
        "ref_wall_s": round(wall, 3),
    }
    if keep_text:
        rec["solution"] = sol.decode()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    ref = RefLib()
    out_path = os.path.join(HERE, "golden.json")
    data = json.load(open(out_path)) if os.path.exists(out_path) else {}
    data.setdefault("_provenance", {
        "generator": "tests/golden/make_golden.py",
        "reference": "oracle/_ref/libegsolve_ref.so built from /root/reference/proj/src by Makefile",
        "fnv": "FNV-1a-64, basis 0xcbf29ce484222325, prime 0x100000001b3, over the text bytes",
    })
    for name, (n, edges, owners) in SPEC_FIXTURES.items():
        a = ref.build(n, edges, owners)
        f, st, wall = ref.solve(a, RefLib.SEQ)
        data[f"spec/{name}"] = summarize(ref, a, f, 1, 0, wall, True)
        data[f"spec/{name}"]["edges"] = edges
        data[f"spec/{name}"]["owners"] = owners
    for inst in SMALL + (BIG if args.big else []):
        kind, p1, p2, W = inst
        key = f"{kind}/{p1}/{p2}/{W}/1"
        t0 = time.time()
        a = ref.fixed(p1, p2, W, 1) if kind == "fixed" else ref.rmat(p1, p2, W, 1)
        workers = 1 if a.m <= 300000 else args.workers
        f, st, wall = ref.solve(a, RefLib.SWEEP, workers=workers)
        data[key] = summarize(ref, a, f, workers, st["rounds"], wall, False)
        print(key, data[key]["tops"], data[key]["solution_fnv"], f"{time.time() - t0:.1f}s", flush=True)
        json.dump(data, open(out_path, "w"), indent=1, sort_keys=True)
    json.dump(data, open(out_path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
