"""Batched k-means++ seeding at cfg2 scale (n=20k, d=80, k=20, 10 restarts): wall time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_03591_b200._device import row_stride  # noqa: E402
from paper_1706_03591_b200.kmeans import _Workspace, batched_kmeanspp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
d, k = 80, 20
g = torch.Generator(device="cuda").manual_seed(0)
blk = torch.zeros((n, row_stride(d)), dtype=torch.float64, device="cuda")
blk[:, :d] = torch.randn((n, d), dtype=torch.float64, device="cuda", generator=g)
ws = _Workspace(blk, d, k)
for rep in range(5):
    kids = np.random.SeedSequence(rep).spawn(10)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    seeds = batched_kmeanspp(ws, kids)
    torch.cuda.synchronize()
    print(f"seeding n={n}: {(time.perf_counter() - t0) * 1e3:.3f} ms")
