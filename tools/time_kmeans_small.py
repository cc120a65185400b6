"""k-means breakdown at cfg2 scale (n=20k, d=80, k=20): seeding vs concurrent Lloyd lanes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import _native  # noqa: E402
from paper_1706_03591_b200._device import ptr, row_stride  # noqa: E402
from paper_1706_03591_b200.kmeans import _Workspace, _lloyd_pool, batched_kmeanspp, run_restarts  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 80
k = int(sys.argv[3]) if len(sys.argv) > 3 else 20
g = torch.Generator(device="cuda").manual_seed(0)
centers = torch.randn((k, d), dtype=torch.float64, device="cuda", generator=g) * 0.3
lab = torch.randint(0, k, (n,), device="cuda", generator=g)
blk = torch.zeros((n, row_stride(d)), dtype=torch.float64, device="cuda")
blk[:, :d] = centers[lab] + torch.randn((n, d), dtype=torch.float64, device="cuda", generator=g) * 0.2
cfg = P.KmeansConfig()
kids = lambda s: np.random.SeedSequence(s).spawn(cfg.restarts)  # noqa: E731
run_restarts(blk, d, k, cfg, kids(0))  # warm (pool, graphs)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run_restarts(blk, d, k, cfg, kids(rep + 1))
    torch.cuda.synchronize()
    t_all = (time.perf_counter() - t0) * 1e3
    pool = _lloyd_pool(n, d, blk.shape[1], k, blk.device)
    ws = pool.ws
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    seeds = batched_kmeanspp(ws, kids(rep + 1))
    torch.cuda.synchronize()
    t_seed = (time.perf_counter() - t0) * 1e3
    iters = []
    for li in range(cfg.restarts):
        iters.append(int(pool.lanes[li].out[1].item()))
    print(f"n={n}: run_restarts {t_all:.2f} ms, seeding {t_seed:.2f} ms, iterations per restart {iters}")
# one lane alone (warm its graph for this workspace first)
lane = pool.lanes[0]
for _ in range(2):
    lane.cent.copy_(seeds[0])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _native.call("csc_kmeans_run", lane.plan, ptr(pool.F), ptr(ws.fnorm), ptr(lane.cent), lane.ldc,
                 ptr(lane.cnorm), ptr(lane.labels), ptr(lane.counts), cfg.max_iters, cfg.tol, ptr(lane.out),
                 None, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
print(f"single lane: {dt:.2f} ms for {int(lane.out[1].item())} iterations -> {dt / max(1, lane.out[1].item()) * 1e3:.1f} us/iter")
