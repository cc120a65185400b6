"""k-means inside a configs[1] dynamic step: seeding vs concurrent Lloyd lanes, iterations."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import _native, generators as G  # noqa: E402
from paper_1706_03591_b200._device import ptr  # noqa: E402
from paper_1706_03591_b200.kmeans import _lloyd_pool, batched_kmeanspp, run_restarts  # noqa: E402

n, k, d = 20000, 20, 80
q1, q2 = G.sbm_probabilities(n, k, 24.0, 0.05)
codes = G.planted_partition_codes(n, k, q1, q2, 7)
labels = np.repeat(np.arange(k), G.block_sizes(n, k))
cfg = P.DynamicConfig(k=k, d=d, p=0.5, filter=P.FilterConfig(order=60))
_, state, _ = P.dynamic_init(G.graph_from_codes(n, codes), cfg, seed=0)
blk = state.features.device_block()
kc = P.KmeansConfig()
for rep in range(4):
    kids = np.random.SeedSequence(rep).spawn(kc.restarts)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run_restarts(blk, d, k, kc, kids)
    torch.cuda.synchronize()
    t_all = (time.perf_counter() - t0) * 1e3
    pool = _lloyd_pool(n, d, blk.shape[1], k, blk.device)
    iters = [int(pool.lanes[i].out[1].item()) for i in range(kc.restarts)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    batched_kmeanspp(pool.ws, kids)
    torch.cuda.synchronize()
    t_seed = (time.perf_counter() - t0) * 1e3
    print(f"run_restarts {t_all:.2f} ms (seeding {t_seed:.2f} ms); iterations {iters}")
lane = pool.lanes[0]
for _ in range(2):
    lane.cent.copy_(batched_kmeanspp(pool.ws, kids)[0])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _native.call("csc_kmeans_run", lane.plan, ptr(pool.F), ptr(pool.ws.fnorm), ptr(lane.cent), lane.ldc,
                 ptr(lane.cnorm), ptr(lane.labels), ptr(lane.counts), kc.max_iters, kc.tol, ptr(lane.out), None,
                 torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
it = int(lane.out[1].item())
print(f"one lane alone: {dt:.2f} ms for {it} iterations -> {dt / max(it, 1) * 1e3:.1f} us/iter")
