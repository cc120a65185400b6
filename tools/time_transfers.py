"""H2D / D2H legs of the e2e apply_filter path at cfg3 size (1M x 128 fp64 = 1 GB)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_03591_b200._device import download_block, upload_block  # noqa: E402

n, d = 1_000_000, 128
src = torch.randn((n, d), dtype=torch.float64).pin_memory()
x_np = src.numpy()
dev = torch.empty((n, d), dtype=torch.float64, device="cuda")
host = torch.empty((n, d), dtype=torch.float64).pin_memory()


def t(fn, reps=4):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return min(ts)


gb = n * d * 8 / 1e9
for name, fn in [("raw pinned H2D", lambda: dev.copy_(src, non_blocking=True)),
                 ("raw pinned D2H", lambda: host.copy_(dev, non_blocking=True)),
                 ("upload_block(pinned numpy)", lambda: upload_block(x_np)),
                 ("download_block", lambda: download_block(dev, d))]:
    ms = t(fn)
    print(f"{name:28s} {ms:8.2f} ms  {gb / ms * 1e3:6.1f} GB/s")
