"""One-shot egs_gpu_solve timing on C4 (dev tool).
usage: python tools/e2e_probe.py [torch] [n_calls]
`torch` first initialises CUDA through torch and runs a few CPU torch ops,
as bench.py does, to expose host-side interference with the upload threads."""
import sys
import time

sys.path.insert(0, ".")
import paper_1710_03647_b200 as egs  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else ""
with_torch = "torch" in mode
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 4
if with_torch:
    import torch
    torch.cuda.set_device(0)
    x = torch.randn(1 << 20)
    for _ in range(10):
        x = x * 1.0001 + 1
    torch.cuda.synchronize()
a = egs.GameArena.fixed(16000000, 16, 100, 1, pinned=True)
out, _o = egs.pinned_empty(a.num_vertices)
opts = egs.SolverOptions(device=0) if "dev" in mode else None
if "ds" in mode:  # a resident context first, as bench.py does
    with egs.DeviceSolver(a, opts) as ds:
        for _ in range(13):
            ds.solve()
for i in range(calls):
    t = time.perf_counter()
    rep = egs.solve(a, options=opts, out=out)
    t1 = time.perf_counter() - t
    g = rep.gpu
    print(f"call {i}: wall {t1*1e3:.1f} ms  upload {g['upload_seconds']*1e3:.1f}  "
          f"solve {g['solve_seconds']*1e3:.1f}  download {g['download_seconds']*1e3:.1f}  "
          f"lib wall {g['wall_seconds']*1e3:.1f}", flush=True)
