import sys, time
sys.path.insert(0, ".")
import paper_1710_03647_b200 as egs
a = egs.GameArena.rmat(22, 16, 100, 1, pinned=True)
out, _o = egs.pinned_empty(a.num_vertices)
for i in range(3):
    t = time.perf_counter()
    rep = egs.solve(a, out=out)
    print(f"call {i}: wall {(time.perf_counter()-t)*1e3:.1f} ms upload {rep.gpu['upload_seconds']*1e3:.1f} solve {rep.gpu['solve_seconds']*1e3:.1f} dl {rep.gpu['download_seconds']*1e3:.1f}", flush=True)
