"""Where does the GPU idle inside a configs[1] dynamic step?  Marker kernels at
phase boundaries + a CUDA-only kernel timeline: idle time between kernels per phase.

Caveat (tools/lane_trace.py): under CUPTI, entering a conditional (while)
graph node shows a ~400 us gap that does not exist in unprofiled runs, so the
k-means lanes' idle time here is overstated."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
import paper_1706_03591_b200.dynamic as D  # noqa: E402
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
_mark_buf = torch.zeros(64, dtype=torch.int32, device="cuda")
NAMES = ["laplacian", "device_signals", "filter_block", "gather_columns", "kmeans"]


def _wrap(mod, name, idx):
    fn = getattr(mod, name)

    def w(*a, **kw):
        _mark_buf[2 * idx:2 * idx + 1].fill_(1)   # marker kernel: phase start
        out = fn(*a, **kw)
        _mark_buf[2 * idx + 1:2 * idx + 2].fill_(2)  # marker kernel: phase end
        return out
    setattr(mod, name, w)


for i, nm in enumerate(NAMES):
    _wrap(D, nm, i)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for gt in graphs[4:]:
        _, state, _ = P.dynamic_step(state, gt, cfg)
    torch.cuda.synchronize()
ev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
            key=lambda e: e.time_range.start)
# kernel intervals merged; markers are the fill kernels on _mark_buf (tiny)
iv = [(e.time_range.start, e.time_range.end, e.name) for e in ev]
steps = len(graphs) - 4
span = (iv[-1][1] - iv[0][0]) / 1e3
merged = []
for s_, e_, _ in iv:
    if merged and s_ <= merged[-1][1]:
        merged[-1][1] = max(merged[-1][1], e_)
    else:
        merged.append([s_, e_])
busy = sum(e - s for s, e in merged) / 1e3
gaps = [(merged[i + 1][0] - merged[i][1], merged[i][1]) for i in range(len(merged) - 1)]
big = sorted(gaps, reverse=True)[:12]
print(f"{steps} steps: kernel span {span / steps:.2f} ms/step, busy {busy / steps:.2f} ms/step, "
      f"idle {(span - busy) / steps:.2f} ms/step in {len(gaps) // steps} gaps/step")


def name_before(t):
    last = None
    for s_, e_, nm in iv:
        if e_ <= t:
            last = nm
    return last


for g, t in big[:6]:
    print(f"  gap {g:8.1f} us after {name_before(t)[:70]}")
# attribute idle to phases: markers are fill kernels on _mark_buf with known order
marks = [(s_, nm) for s_, e_, nm in iv if "FillFunctor<int>" in nm]
phase_of = []
order = []
for i_, nm in enumerate(NAMES):
    order += [nm + ":in", nm + ":after"]
# walk markers in time; every marker toggles to the next label in the per-step sequence
labels_seq = []
seq = ["laplacian", "device_signals", "filter_block", "gather_columns", "gather_columns", "kmeans"]
idle_by = {}
cur_label = "step-start"
mi = 0
mk = [s_ for s_, nm in marks]
for (gsz, gt) in gaps:
    # label = last marker before the gap start
    last = None
    for s_, e_, nm in iv:
        if e_ > gt:
            break
        if "FillFunctor<int>" in nm:
            last = s_
    idle_by.setdefault(last, 0.0)
    idle_by[last] += gsz
print(f"  markers per step: {len(marks) // steps}")
tot = 0.0
rows = []
for idx, (s_, nm) in enumerate(marks):
    v = idle_by.get(s_, 0.0)
    rows.append((idx % (len(marks) // steps), v))
acc = {}
for pos, v in rows:
    acc[pos] = acc.get(pos, 0.0) + v / 1e3 / steps
for pos in sorted(acc):
    print(f"  after marker #{pos}: idle {acc[pos]:.3f} ms/step")
