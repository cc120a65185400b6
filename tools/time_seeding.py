"""Batched k-means++ seeding (csc_kmeanspp_batch) wall time on random features.

    python tools/time_seeding.py [n] [d] [k] [restarts]     (default 20000 80 20 10)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_03591_b200._device import row_stride  # noqa: E402
from paper_1706_03591_b200.kmeans import _Workspace, batched_kmeanspp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 80
k = int(sys.argv[3]) if len(sys.argv) > 3 else 20
R = int(sys.argv[4]) if len(sys.argv) > 4 else 10
g = torch.Generator(device="cuda").manual_seed(0)
blk = torch.zeros((n, row_stride(d)), dtype=torch.float64, device="cuda")
blk[:, :d] = torch.randn((n, d), dtype=torch.float64, device="cuda", generator=g)
ws = _Workspace(blk, d, k)
out = None
for rep in range(4):
    kids = np.random.SeedSequence(7).spawn(R)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    seeds = batched_kmeanspp(ws, kids)
    torch.cuda.synchronize()
    print(f"seeding n={n} d={d} k={k} R={R}: {(time.perf_counter() - t0) * 1e3:.3f} ms", flush=True)
    out = seeds.cpu().numpy()
np.save(os.environ.get("SEEDS_OUT", "/tmp/seeds.npy"), out)
