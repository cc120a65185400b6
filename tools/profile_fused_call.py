"""Kernel timeline (CUPTI via torch.profiler) of one fused kmeans() call on a configs[1] Theta."""
import importlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from dyn_kmeans_probe import sequence  # noqa: E402

KM = importlib.import_module("paper_1706_03591_b200.kmeans")
D = importlib.import_module("paper_1706_03591_b200.dynamic")
graphs = sequence(3)
cfg = P.DynamicConfig(k=20, d=80, p=0.5, filter=P.FilterConfig(order=60))
captured = []
orig = KM._kmeans_prepared


def spy(theta, d, k, kcfg, children, draws):
    captured.append((theta.clone(), children, draws))
    return orig(theta, d, k, kcfg, children, draws)


D._kmeans_prepared = spy
_, state, _ = P.dynamic_init(graphs[0], cfg, seed=0)
for gt in graphs[1:]:
    _, state, _ = P.dynamic_step(state, gt, cfg)
theta, children, draws = captured[-1]
for rep in range(3):
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        KM.run_restarts(theta, 80, 20, cfg.kmeans, children, draws)
        torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
for e in evs:
    print(f"{(e.time_range.start - t0):9.1f} us  dur {e.time_range.elapsed_us():8.1f}  {e.name[:90]}")
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU]
print("host span (first CPU event to last):", max(e.time_range.end for e in cpu) - min(e.time_range.start for e in cpu), "us")
