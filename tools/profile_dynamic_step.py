"""Kernel timeline of one configs[1] dynamic step (torch.profiler / CUPTI): per-kernel totals and GPU idle gaps."""
import collections

import numpy as np
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from dyn_kmeans_probe import sequence  # noqa: E402

graphs = sequence(5)
cfg = P.DynamicConfig(k=20, d=80, p=0.5, filter=P.FilterConfig(order=60))
_, state, _ = P.dynamic_init(graphs[0], cfg, seed=0)
for gt in graphs[1:4]:
    _, state, _ = P.dynamic_step(state, gt, cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ph = {}
    _, state, _ = P.dynamic_step(state, graphs[4], cfg, timings=ph)
    torch.cuda.synchronize()
print("phases (host ms):", {k: round(v, 3) for k, v in ph.items()})
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
tot = collections.defaultdict(lambda: [0, 0.0])
busy_end, gaps = t0, 0.0
for e in evs:
    tot[e.name[:70]][0] += 1
    tot[e.name[:70]][1] += e.time_range.elapsed_us()
    if e.time_range.start > busy_end:
        gaps += e.time_range.start - busy_end
    busy_end = max(busy_end, e.time_range.end)
print(f"GPU span {busy_end - t0:.1f} us, idle gaps {gaps:.1f} us")
for name, (c, us) in sorted(tot.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{us:9.1f} us  x{c:4d}  {name}")
print("gaps > 15 us (after kernel -> before kernel):")
prev = None
for e in evs:
    if prev is not None and e.time_range.start - prev.time_range.end > 15:
        print(f"  {e.time_range.start - prev.time_range.end:7.1f} us  after {prev.name[:50]}  before {e.name[:50]}")
    if prev is None or e.time_range.end > prev.time_range.end:
        prev = e
sw = [e for e in evs if "sweep_kernel" in e.name]
gaps = [b.time_range.start - a.time_range.end for a, b in zip(sw, sw[1:])]
if gaps:
    print(f"sweeps: {len(sw)}, mean duration {np.mean([e.time_range.elapsed_us() for e in sw]):.1f} us, "
          f"gap between consecutive sweeps median {np.median(gaps):.1f} us, total gaps {np.sum(gaps):.0f} us")
