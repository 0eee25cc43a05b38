"""Randomised GPU-vs-oracle stress run (dev tool, test infrastructure: it
loads the oracle).  usage: python tools/stress.py [seconds] [seed0]
Random arenas of varied size, degree, weight range and bias, every mode, with
and without the certificate, 4- and 8-byte records; any mismatch is printed
with its reproduction parameters and the run exits non-zero."""
import os
import random
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1710_03647_b200 as egs  # noqa: E402
from oracle_bindings import Oracle  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
oracle = Oracle()
t0 = time.time()
cases = bad = 0
k = seed0
while time.time() - t0 < budget:
    r = random.Random(k)
    n = r.choice([1, 2, 5, 33, 100, 300, 1000, 3000])
    maxdeg = r.choice([1, 2, 4, 8, 40, 120])
    W = r.choice([1, 3, 10, 100, 1000, 10 ** 6])
    bias = r.choice([0, 0, -1, 1])
    owners = [r.randint(0, 1) for _ in range(n)]
    edges = []
    for v in range(n):
        for _ in range(r.randint(1, maxdeg)):
            edges.append((v, r.randrange(n), r.randint(-W, W) + bias * r.randint(0, max(1, W // 4))))
    if r.random() < 0.2 and n > 10:  # a hub column and row
        h = r.randrange(n)
        edges += [(h, r.randrange(n), r.randint(-W, W)) for _ in range(5000)]
        edges += [(r.randrange(n), h, r.randint(-W, W)) for _ in range(5000)]
    r.shuffle(edges)
    a = egs.GameArena.build(n, edges, owners)
    g = oracle.build(n, edges, owners)
    want, _ = oracle.solve_seq(g)
    wide = r.random() < 0.3
    if wide:
        os.environ["EGS_EDGE_FORMAT"] = "8"
    else:
        os.environ.pop("EGS_EDGE_FORMAT", None)
    for mode in ("auto", "dense", "sparse"):
        for certify in (True, False):
            ci = r.choice([1, 2, 5])
            rep = egs.solve(a, options=egs.SolverOptions(mode=mode, certify=certify,
                                                         cert_interval=ci))
            cases += 1
            if not np.array_equal(rep.measure, want):
                bad += 1
                print(f"MISMATCH seed={k} n={n} maxdeg={maxdeg} W={W} bias={bias} "
                      f"mode={mode} certify={certify} ci={ci} wide={wide}", flush=True)
    k += 1
print(f"stress: {cases} solves over {k - seed0} arenas, {bad} mismatches, "
      f"{time.time() - t0:.0f} s", flush=True)
sys.exit(1 if bad else 0)
