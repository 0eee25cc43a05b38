# compute-sanitizer over small solves (memcheck, racecheck, synccheck)
S=/usr/local/cuda/bin/compute-sanitizer
cat > /tmp/san_target.py <<'PY'
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import paper_1710_03647_b200 as egs
from arena_gen import random_arena
a = egs.GameArena.fixed(3000, 4, 100, 1)
for mode in ("auto", "dense", "sparse"):
    with egs.DeviceSolver(a, egs.SolverOptions(mode=mode)) as ds:
        ds.solve(); f = ds.read_measure(); ds.write_solution(); assert ds.is_fixpoint(f)
h = egs.GameArena.rmat(10, 16, 100, 1)
egs.solve(h)
for seed in range(5):
    n, e, o = random_arena(seed, max_n=30, max_deg=5)
    egs.solve(egs.GameArena.build(n, e, o))
# the chunked transpose (default only for >= 2^27 edges), the flat long-row
# relabel (R-MAT hubs), the host-pool narrowing / widening (>= 2^20), two
# ranks (SAN_LIGHT=1: the solve kernel on the small arenas above only)
import os
if os.environ.get("SAN_LIGHT"):
    print("sanitizer target ok")
    sys.exit(0)
os.environ["EGS_CSC_SORT"] = "inc"
for arena in (egs.GameArena.rmat(12, 16, 100, 1), egs.GameArena.fixed(20000, 8, 100, 1)):
    with egs.DeviceSolver(arena, egs.SolverOptions(debug_checks=True)) as ds:
        ds.solve()
del os.environ["EGS_CSC_SORT"]
if os.environ.get("SAN_BIG"):  # (memcheck only: slow under the sanitizer)
    r = egs.solve(egs.GameArena.fixed(1100000, 1, 100, 1))
# two ranks of the device exchange in one process
from paper_1710_03647_b200.distributed import solve_local
reps, parts = solve_local(egs.GameArena.fixed(3000, 4, 100, 1), 2,
                          options=egs.SolverOptions(device=0))
assert np.array_equal(reps[0].measure, reps[1].measure)
for p_ in parts:
    p_.close()
print("sanitizer target ok")
PY
for tool in ${SAN_TOOLS:-memcheck racecheck synccheck initcheck}; do
  echo "== $tool"
  big=""; [ $tool = memcheck ] && big=1
  SAN_BIG=$big timeout 700 $S --tool $tool --print-limit 20 python /tmp/san_target.py 2>&1 | tail -6
done
