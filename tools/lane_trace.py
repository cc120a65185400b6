"""Kernel-by-kernel timeline of ONE restart lane's csc_kmeans_run graph (CUPTI)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1706_03591_b200 import _native  # noqa: E402
from paper_1706_03591_b200._device import ptr, row_stride  # noqa: E402
from paper_1706_03591_b200.kmeans import KmeansConfig, _lloyd_pool, batched_kmeanspp, run_restarts  # noqa: E402

n, d, k = 20000, 80, 20
g = torch.Generator(device="cuda").manual_seed(0)
blk = torch.zeros((n, row_stride(d)), dtype=torch.float64, device="cuda")
blk[:, :d] = torch.randn((n, d), dtype=torch.float64, device="cuda", generator=g)
cfg = KmeansConfig(max_iters=8)
run_restarts(blk, d, k, cfg, np.random.SeedSequence(0).spawn(2))
pool = _lloyd_pool(n, d, blk.shape[1], k, blk.device)
seeds = batched_kmeanspp(pool.ws, np.random.SeedSequence(1).spawn(1))
lane = pool.lanes[0]
for it in range(2):
    lane.cent.copy_(seeds[0])
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        _native.call("csc_kmeans_run", lane.plan, ptr(pool.F), ptr(pool.ws.fnorm), ptr(lane.cent), lane.ldc,
                     ptr(lane.cnorm), ptr(lane.labels), ptr(lane.counts), cfg.max_iters, float(cfg.tol),
                     ptr(lane.out), None, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
ev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
            key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = t0
for e in ev:
    gap = e.time_range.start - prev_end
    print(f"{(e.time_range.start - t0):8.1f} us  +gap {gap:7.1f}  dur {e.time_range.end - e.time_range.start:6.1f}  {e.name[:60]}")
    prev_end = max(prev_end, e.time_range.end)
print("iterations:", int(lane.out[1].item()))
