"""cProfile of the host side of configs[1] dynamic steps (top cumulative entries)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import generators as G  # noqa: E402

n, k, d = 20000, 20, 80
q1, q2 = G.sbm_probabilities(n, k, 24.0, 0.05)
codes = G.planted_partition_codes(n, k, q1, q2, 7)
labels = np.repeat(np.arange(k), G.block_sizes(n, k))
graphs = [G.graph_from_codes(n, codes)]
cur = codes
for t in range(1, 12):
    dn, inn, labels = G.node_switch(cur, n, labels, k, q1, q2, 0.005, seed=200 + t)
    cur = np.union1d(np.setdiff1d(cur, dn, assume_unique=True), inn)
    dl, il = G.edge_churn(cur, n, labels, q1, q2, 0.01, seed=100 + t)
    graphs.append(graphs[-1].apply_delta(dn, inn).apply_delta(dl, il))
    cur = np.union1d(np.setdiff1d(cur, dl, assume_unique=True), il)
cfg = P.DynamicConfig(k=k, d=d, p=0.5, filter=P.FilterConfig(order=60))
_, state, _ = P.dynamic_init(graphs[0], cfg, seed=0)
for gt in graphs[1:4]:
    _, state, _ = P.dynamic_step(state, gt, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for gt in graphs[4:]:
    _, state, _ = P.dynamic_step(state, gt, cfg)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(22)
