"""Where a configs[4]-shape k-means call spends its GPU time (tools only).

    python tools/kmeans_cfg5_profile.py [--restarts 10] [--what cfg5|cfg3]

Builds the features of a cfg5 (or cfg3) static pipeline (moment bisection at
the BASELINE order), then times P.kmeans(features, k) and prints per-kernel
totals from torch.profiler (CUPTI records the kernels inside the lanes' CUDA
graphs) plus the iterations of every restart.
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import generators as G  # noqa: E402
from paper_1706_03591_b200.filters import FilteredBlock, _search_cutoff  # noqa: E402
from paper_1706_03591_b200.signals import device_signals  # noqa: E402
import importlib  # noqa: E402
K = importlib.import_module("paper_1706_03591_b200.kmeans")

ap = argparse.ArgumentParser()
ap.add_argument("--restarts", type=int, default=10)
ap.add_argument("--what", default="cfg5")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
if a.what == "cfg5":
    n, k, d, m, deg, ratio = 2_000_000, 64, 96, 80, 20.0, 0.05
else:
    n, k, d, m, deg, ratio = 1_000_000, 100, 128, 100, 32.0, 0.02
q1, q2 = G.sbm_probabilities(n, k, deg, ratio)
lap = P.laplacian(G.graph_from_codes(n, G.planted_partition_codes(n, k, q1, q2, 5)))
blk = device_signals(n, d, 0)
cut, filt, poly, iters, est = _search_cutoff(lap, k, FilteredBlock(blk, d), (0.0, 2.0), P.FilterConfig(order=m),
                                             None, 1.0)
feats = P.FeatureMatrix._from_block(filt.blk, d, np.zeros(d, np.int64), np.arange(d))
del blk
torch.cuda.empty_cache()
cfg = P.KmeansConfig(restarts=a.restarts)
for rep in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    asg = P.kmeans(feats, k, cfg, seed=rep)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    pool = K._LLOYD_POOL
    its = [int(pool.lanes[i].out[1].item()) for i in range(min(a.restarts, len(pool.lanes)))] if pool else []
    print(f"kmeans {ms:.1f} ms, iterations per restart {its} (sum {sum(its)}), cost {asg.feature_cost:.6f}",
          flush=True)
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    P.kmeans(feats, k, cfg, seed=7)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
