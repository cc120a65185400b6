"""Whole k-means (10 restarts, device loop lanes) at cfg3 scale with different assign tiles."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import _native  # noqa: E402
from paper_1706_03591_b200._device import row_stride  # noqa: E402

n, d, k = 1_000_000, 128, 100
if os.environ.get("BLOBS"):
    g = torch.Generator(device="cuda").manual_seed(0)
    centers = torch.randn((k, d), dtype=torch.float64, device="cuda", generator=g) * 0.3
    lab = torch.randint(0, k, (n,), device="cuda", generator=g)
    blk = torch.zeros((n, row_stride(d)), dtype=torch.float64, device="cuda")
    blk[:, :d] = centers[lab] + torch.randn((n, d), dtype=torch.float64, device="cuda", generator=g) * 0.25
else:  # the cfg3 pipeline's features (tools/time_pipeline.py --what cfg3)
    from paper_1706_03591_b200 import generators as G
    from paper_1706_03591_b200.filters import FilteredBlock, _search_cutoff
    from paper_1706_03591_b200.signals import device_signals
    q1, q2 = G.sbm_probabilities(n, k, 32.0, 0.02)
    lap = P.laplacian(G.graph_from_codes(n, G.planted_partition_codes(n, k, q1, q2, 3)))
    x = device_signals(n, d, 0)
    _, filt, _, _, _ = _search_cutoff(lap, k, FilteredBlock(x, d), (0.0, 2.0), P.FilterConfig(order=100), None, 1.0)
    blk = filt.blk
lib = _native.lib()
for tile in sys.argv[1:] or ["88", "0"]:
    _native.check(lib.csc_kmeans_tuning(b"assign_tile", int(tile)), "tuning")
    P.kmeans((blk, d), k, P.KmeansConfig(restarts=2, max_iters=3), seed=9)  # warm (pool, graphs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    asg = P.kmeans((blk, d), k, P.KmeansConfig(), seed=1)
    torch.cuda.synchronize()
    print(f"tile {tile}: kmeans {(time.perf_counter() - t0) * 1e3:.1f} ms, cost {asg.feature_cost:.9f}")
_native.check(lib.csc_kmeans_tuning(b"assign_tile", 0), "tuning")
