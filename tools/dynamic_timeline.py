"""GPU busy time vs wall time of cfg2 dynamic steps (torch.profiler / CUPTI kernel intervals)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import generators as G  # noqa: E402

n, k, d = 20000, 20, 80
q1, q2 = G.sbm_probabilities(n, k, 24.0, 0.05)
codes = G.planted_partition_codes(n, k, q1, q2, 7)
labels = np.repeat(np.arange(k), G.block_sizes(n, k))
graphs = [G.graph_from_codes(n, codes)]
cur = codes
for t in range(1, 8):
    dn, inn, labels = G.node_switch(cur, n, labels, k, q1, q2, 0.005, seed=200 + t)
    cur = np.union1d(np.setdiff1d(cur, dn, assume_unique=True), inn)
    dl, il = G.edge_churn(cur, n, labels, q1, q2, 0.01, seed=100 + t)
    graphs.append(graphs[-1].apply_delta(dn, inn).apply_delta(dl, il))
    cur = np.union1d(np.setdiff1d(cur, dl, assume_unique=True), il)
cfg = P.DynamicConfig(k=k, d=d, p=0.5, filter=P.FilterConfig(order=60))
_, state, _ = P.dynamic_init(graphs[0], cfg, seed=0)
for gt in graphs[1:4]:
    _, state, _ = P.dynamic_step(state, gt, cfg)
import paper_1706_03591_b200.dynamic as D  # noqa: E402
from torch.profiler import record_function  # noqa: E402


def _wrap(mod, name):
    fn = getattr(mod, name)

    def w(*a, **kw):
        with record_function("phase:" + name):
            return fn(*a, **kw)
    setattr(mod, name, w)


for _nm in ("laplacian", "device_signals", "filter_block", "gather_columns", "kmeans", "_search_cutoff"):
    if hasattr(D, _nm):
        _wrap(D, _nm)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    for gt in graphs[4:]:
        _, state, _ = P.dynamic_step(state, gt, cfg)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
allev = prof.events()
ev = [e for e in allev if e.device_type == torch.autograd.DeviceType.CUDA]
ranges = [e for e in allev if e.name.startswith("phase:")]
iv = sorted((e.time_range.start, e.time_range.end) for e in ev)
busy, cs, ce = 0.0, None, None
for s, e in iv:
    if cs is None or s > ce:
        if cs is not None:
            busy += ce - cs
        cs, ce = s, e
    else:
        ce = max(ce, e)
if cs is not None:
    busy += ce - cs
span = (iv[-1][1] - iv[0][0]) / 1e3 if iv else 0.0
steps = len(graphs) - 4
merged = []
for s_, e_ in iv:
    if merged and s_ <= merged[-1][1]:
        merged[-1][1] = max(merged[-1][1], e_)
    else:
        merged.append([s_, e_])


def busy_in(t0, t1):
    tot = 0.0
    for s_, e_ in merged:
        a_, b_ = max(s_, t0), min(e_, t1)
        if b_ > a_:
            tot += b_ - a_
    return tot


agg = {}
for r in ranges:
    t0_, t1_ = r.time_range.start, r.time_range.end
    a = agg.setdefault(r.name, [0.0, 0.0])
    a[0] += (t1_ - t0_) / 1e3
    a[1] += busy_in(t0_, t1_) / 1e3
for nm, (w_, b_) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"  {nm:24s} host {w_ / (len(graphs) - 4):7.3f} ms/step, GPU busy inside {b_ / (len(graphs) - 4):7.3f} ms/step")
print(f"{steps} steps: wall {wall / steps:.2f} ms/step, GPU busy (union of kernels) {busy / 1e3 / steps:.2f} ms/step, "
      f"kernel span {span / steps:.2f} ms/step, {len(ev) // steps} device events/step")
