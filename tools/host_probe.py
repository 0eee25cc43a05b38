"""Host-side bandwidth probe for the e2e path (dev tool): pinned H2D
bandwidth, host memory read bandwidth with 16 threads, then one-shot solves
of C4 with the library's upload timeline (EGS_VERBOSE)."""
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
x = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
d = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for _ in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    d.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    print(f"H2D pinned 1 GiB: {1.0737 / (time.perf_counter() - t):.1f} GB/s", flush=True)
a = np.ones(1 << 28, dtype=np.int64)  # 2 GiB
def work(lo, hi, out, k):
    out[k] = int(a[lo:hi].sum())
for T in (1, 8, 16):
    out = [0] * T
    t = time.perf_counter()
    th = [threading.Thread(target=work, args=(len(a) * k // T, len(a) * (k + 1) // T, out, k))
          for k in range(T)]
    [h.start() for h in th]
    [h.join() for h in th]
    print(f"host read 2 GiB, {T} threads: {2.147 / (time.perf_counter() - t):.1f} GB/s", flush=True)
