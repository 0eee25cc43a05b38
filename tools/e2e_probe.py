import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1710_03647_b200 as egs
a = egs.GameArena.fixed(16000000, 16, 100, 1, pinned=True)
out, _o = egs.pinned_empty(a.num_vertices)
for i in range(4):
    t = time.perf_counter()
    rep = egs.solve(a, out=out)
    t1 = time.perf_counter() - t
    g = rep.gpu
    print(f"call {i}: wall {t1*1e3:.1f} ms  upload {g['upload_seconds']*1e3:.1f}  solve {g['solve_seconds']*1e3:.1f}  download {g['download_seconds']*1e3:.1f}  lib wall {g['wall_seconds']*1e3:.1f}", flush=True)
