"""Whole k-means on real cfg5 features with different restart-lane widths (CSC_KMEANS_LANES)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import generators as G  # noqa: E402
from paper_1706_03591_b200.filters import FilteredBlock, _search_cutoff  # noqa: E402
from paper_1706_03591_b200.signals import device_signals  # noqa: E402

n, k, d, m = 2_000_000, 64, 96, 80
q1, q2 = G.sbm_probabilities(n, k, 20.0, 0.05)
lap = P.laplacian(G.graph_from_codes(n, G.planted_partition_codes(n, k, q1, q2, 5)))
_, filt, _, _, _ = _search_cutoff(lap, k, FilteredBlock(device_signals(n, d, 0), d), (0.0, 2.0),
                                  P.FilterConfig(order=m), None, 1.0)
blk = filt.blk
P.kmeans((blk, d), k, P.KmeansConfig(restarts=2, max_iters=3), seed=9)  # warm
for w in sys.argv[1:] or ["10", "2", "1"]:
    os.environ["CSC_KMEANS_LANES"] = w
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    asg = P.kmeans((blk, d), k, P.KmeansConfig(), seed=1)
    torch.cuda.synchronize()
    print(f"lanes {w}: kmeans {(time.perf_counter() - t0) * 1e3:.1f} ms, cost {asg.feature_cost:.9f}")
