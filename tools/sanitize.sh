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
print("sanitizer target ok")
PY
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 900 $S --tool $tool --print-limit 20 python /tmp/san_target.py 2>&1 | tail -6
done
