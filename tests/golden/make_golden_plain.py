"""Certificate-free digests of the full-size BASELINE configs, computed on the
GPU by PLAIN value iteration (SolverOptions(certify=False)): the reference's
own iteration (lift measure_ops.hpp:32-52 from f = 0 up to credit_cap,
solver_par.cpp:126-245 / :247-435) with no losing-region certificate, so the
losing vertices climb O(W) per round all the way to credit_cap (~10^6 rounds
on C4).  It shares no code with the certificate, so agreement of
the two digests pins the certified solve on inputs where the CPU reference
cannot finish (C4: ~17 days of sweeps projected).

Run on the GPU box (needs the built library):

    python tests/golden/make_golden_plain.py --out gpurun_out/golden_plain.json C4,C3,F16

For every config it first times a bounded probe (--probe rounds) and prints
it, then runs the full plain solve with a device-side timeout of --budget
seconds.  It records the write_solution digest of the plain measure
(SHA-256, FNV-1a-64, length, tops, finite sum / max), the plain run's rounds
and time, and whether the certified solve gave the identical bytes.
tests/golden/golden.json stores these under "plain_gpu" of each config key;
tests/test_gpu_parity.py::test_full_size_golden checks the certified GPU
output against them (and against the reference's own digests where the
reference finished: C2, C5, F16, C3).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import numpy as np  # noqa: E402

import paper_1710_03647_b200 as egs  # noqa: E402

INT64_MAX = np.iinfo(np.int64).max
CONFIGS = {"C4": ("fixed", (16_000_000, 16, 100)), "C3": ("rmat", (22, 16, 100)),
           "F16": ("fixed", (1_000_000, 16, 100)), "C2": ("fixed", (1_000_000, 8, 1000)),
           "C5": ("fixed", (1_000_000, 8, 100_000)), "C1": ("fixed", (10_000, 4, 100))}


def digest(sol: bytes, f: np.ndarray) -> dict:
    fin = f[f != INT64_MAX]
    return {"solution_bytes": len(sol), "solution_sha256": hashlib.sha256(sol).hexdigest(),
            "tops": int((f == INT64_MAX).sum()), "sum_finite": int(fin.sum()),
            "max_finite": int(fin.max()) if fin.size else 0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--probe", type=int, default=4000, help="rounds of the timing probe")
    ap.add_argument("--budget", type=float, default=2400.0, help="max projected seconds per config")
    ap.add_argument("--mode", default="sweep",
                    help="sweep: in-place rounds, the reference's solve_sweep (fewest rounds)")
    ap.add_argument("configs", nargs="?", default="C4,C3,F16")
    args = ap.parse_args()
    out = {}
    if os.path.exists(args.out):
        with open(args.out) as fh:
            out = json.load(fh)
    for cfg in args.configs.split(","):
        gen, gargs = CONFIGS[cfg]
        key = f"{gen}/" + "/".join(map(str, gargs)) + "/1"
        if key in out and "plain_gpu" in out[key]:
            continue
        a = getattr(egs.GameArena, gen)(*gargs, 1)
        rec = {"config": cfg, "n": a.num_vertices, "m": a.num_edges}
        # certified solve (the product path)
        with egs.DeviceSolver(a) as ds:
            st = ds.solve()
            f_cert = ds.read_measure()
            sol_cert = ds.write_solution().encode()
        rec["certified"] = digest(sol_cert, f_cert)
        rec["certified"]["rounds"] = int(st.rounds)
        # probe: bounded plain rounds -> seconds per round
        opts = dict(certify=False, mode=args.mode)
        with egs.DeviceSolver(a, egs.SolverOptions(**opts, sweep_bound=args.probe)) as ds:
            t0 = time.time()
            try:
                ds.solve()
                probe_done = True
            except egs.BoundExhaustedError:
                probe_done = False
            dt = time.time() - t0
        print(f"{cfg}: probe {args.probe} rounds in {dt:.2f} s (finished={probe_done})", flush=True)
        with egs.DeviceSolver(a, egs.SolverOptions(**opts, timeout_seconds=args.budget)) as ds:
            t0 = time.time()
            try:
                st = ds.solve()
            except egs.TimeoutError_ as e:
                rec["plain_gpu"] = {"status": f"timeout after {args.budget} s: {e}"}
                print(cfg, rec, flush=True)
                out[key] = {**out.get(key, {}), **rec}
                continue
            wall = time.time() - t0
            f_plain = ds.read_measure()
            assert ds.is_fixpoint(f_plain)
            sol_plain = ds.write_solution().encode()
        p = digest(sol_plain, f_plain)
        p.update(rounds=int(st.rounds), dense_rounds=int(st.dense_rounds),
                 sparse_rounds=int(st.sparse_rounds), solve_s=round(float(st.solve_seconds), 3),
                 wall_s=round(wall, 3), edges_relaxed=int(st.edges_relaxed),
                 solver=f"GPU plain value iteration (certify=False, mode={args.mode})")
        rec["plain_gpu"] = p
        rec["certified_equals_plain"] = bool(sol_plain == sol_cert)
        print(cfg, json.dumps(rec), flush=True)
        out[key] = {**out.get(key, {}), **rec}
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1, sort_keys=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
