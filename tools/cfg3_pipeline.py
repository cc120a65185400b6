"""Phase times of the configs[2] pipeline (csc_assign's steps, tools only):
device signals, moment bisection for lambda_100 (resident orders when they
fit), k-means k=100 x 10 restarts (lane path: tensor-core screen, exact sums).

    python tools/cfg3_pipeline.py [--calls 3]
"""
import argparse
import importlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import generators as G  # noqa: E402
from paper_1706_03591_b200.filters import FilteredBlock, _search_cutoff  # noqa: E402
from paper_1706_03591_b200.signals import device_signals  # noqa: E402

KM = importlib.import_module("paper_1706_03591_b200.kmeans")
ap = argparse.ArgumentParser()
ap.add_argument("--calls", type=int, default=3)
a = ap.parse_args()
w = bench.WORKLOADS["cfg3"]
codes, _ = bench.make_graph_codes(w)
lap = P.laplacian(G.graph_from_codes(w["n"], codes))
k, d = w["k"], w["d"]
cfg = P.FilterConfig(order=w["order"])


def now():
    torch.cuda.synchronize()
    return time.perf_counter()


for c in range(a.calls):
    t0 = now()
    blk = device_signals(lap.n, d, np.random.SeedSequence(c).spawn(2)[0])
    t1 = now()
    cut, filt, poly, iters, est = _search_cutoff(lap, k, FilteredBlock(blk, d), (0.0, lap.lambda_max_bound), cfg,
                                                 None, 1.0)
    t2 = now()
    fblk = filt.blk
    kids = np.random.SeedSequence(c).spawn(2)[1].spawn(10)
    labels, cost2 = KM.run_restarts(fblk, d, k, P.KmeansConfig(), kids)
    t3 = now()
    its = [int(l.out[1].item()) if l.out.numel() > 1 else -1 for l in KM._LLOYD_POOL.lanes[:10]]
    print(f"call {c}: signals {(t1 - t0) * 1e3:.1f} ms, bisection {(t2 - t1) * 1e3:.1f} ms ({iters} probes), "
          f"k-means {(t3 - t2) * 1e3:.1f} ms (lane iterations {its}), total {(t3 - t0) * 1e3:.1f} ms", flush=True)
