"""Host time of the restart-lane launches inside run_restarts (no sync between them)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_03591_b200 import _native  # noqa: E402
from paper_1706_03591_b200._device import ptr, row_stride  # noqa: E402
from paper_1706_03591_b200.kmeans import KmeansConfig, _lloyd_pool, batched_kmeanspp, run_restarts  # noqa: E402

n, d, k = 20000, 80, 20
g = torch.Generator(device="cuda").manual_seed(0)
blk = torch.zeros((n, row_stride(d)), dtype=torch.float64, device="cuda")
blk[:, :d] = torch.randn((n, d), dtype=torch.float64, device="cuda", generator=g)
cfg = KmeansConfig()
run_restarts(blk, d, k, cfg, np.random.SeedSequence(0).spawn(10))
pool = _lloyd_pool(n, d, blk.shape[1], k, blk.device)
seeds = batched_kmeanspp(pool.ws, np.random.SeedSequence(1).spawn(10))
torch.cuda.synchronize()
for rep in range(3):
    ts = []
    for li in range(10):
        lane = pool.lanes[li]
        t0 = time.perf_counter()
        with torch.cuda.stream(lane.stream):
            lane.cent.copy_(seeds[li])
        t1 = time.perf_counter()
        _native.call("csc_kmeans_run", lane.plan, ptr(pool.F), ptr(pool.ws.fnorm), ptr(lane.cent), lane.ldc,
                     ptr(lane.cnorm), ptr(lane.labels), ptr(lane.counts), cfg.max_iters, float(cfg.tol),
                     ptr(lane.out), None, lane.stream.cuda_stream)
        t2 = time.perf_counter()
        ts.append(((t1 - t0) * 1e6, (t2 - t1) * 1e6))
    torch.cuda.synchronize()
    print("per lane host us (seed copy, csc_kmeans_run):", [(round(a), round(b)) for a, b in ts])
