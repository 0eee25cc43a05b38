"""Where the end-to-end one-shot solve (egs_gpu_solve) spends its time, next
to the raw PCIe copy floor (dev tool).  python tools/e2e_breakdown.py [C4]"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1710_03647_b200 as egs  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
kind, args = CONFIGS[cfg]
a = getattr(egs.GameArena, kind)(*args, 1, pinned=True)
n = a.num_vertices
out, _own = egs.pinned_empty(n)
for _ in range(2):
    egs.solve(a, out=out)
for _ in range(5):
    t = time.perf_counter()
    r = egs.solve(a, out=out)
    w = time.perf_counter() - t
    g = r.gpu
    print(f"wall {w*1e3:.2f} ms  upload {g['upload_seconds']*1e3:.2f}  solve {g['solve_seconds']*1e3:.2f}"
          f"  download {g['download_seconds']*1e3:.2f}  rest {(w - g['upload_seconds'] - g['solve_seconds'] - g['download_seconds'])*1e3:.2f}",
          flush=True)
# raw copy floor: the same byte counts, pinned, one stream
for nbytes, d in ((1_424_000_008, "h2d"), (n * 8, "d2h")):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dv = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        t = time.perf_counter()
        if d == "h2d":
            dv.copy_(h, non_blocking=True)
        else:
            h.copy_(dv, non_blocking=True)
        torch.cuda.synchronize()
        s = time.perf_counter() - t
    print(f"raw {d} {nbytes/1e6:.0f} MB: {s*1e3:.2f} ms = {nbytes/s/1e9:.1f} GB/s", flush=True)
    del h, dv
