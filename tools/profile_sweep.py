"""Short cfg3 run for ncu: build the graph, filter a few orders (fp64 or fp32).

    python tools/profile_sweep.py [--precision fp32] [--orders 6] [--d 128]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import generators as G  # noqa: E402
from paper_1706_03591_b200._device import row_stride  # noqa: E402
from paper_1706_03591_b200.filters import filter_block  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--precision", default="fp64")
ap.add_argument("--orders", type=int, default=6)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--workload", default="cfg3")
a = ap.parse_args()
if a.workload == "cfg3":
    n, k, deg, ratio = 1_000_000, 100, 32.0, 0.02
    q1, q2 = G.sbm_probabilities(n, k, deg, ratio)
    g = G.graph_from_codes(n, G.planted_partition_codes(n, k, q1, q2, 3))
else:  # cfg4 skewed
    n = 4_000_000
    cache = "/tmp/csc_cfg4_codes.npy"  # tool-side cache only (tests/bench never read it)
    if os.path.exists(cache):
        g = G.graph_from_codes(n, np.load(cache))
    else:
        g, _ = G.chung_lu_sbm(n, 50, 16.0, 2.3, 20000.0, 0.05, seed=4)
        np.save(cache, g.edge_i * n + g.edge_j)
lap = P.laplacian(g)
dt = torch.float64 if a.precision == "fp64" else torch.float32
ld = row_stride(a.d, dt)
blk = torch.zeros((n, ld), dtype=dt, device="cuda")
blk[:, :a.d] = torch.randn((n, a.d), dtype=dt, device="cuda") / np.sqrt(a.d)
poly = P.cheb_coeffs(0.05, 2.0, a.orders)
out = torch.empty_like(blk)
work = torch.empty((2 * n, ld), dtype=dt, device="cuda")
for _ in range(2):
    filter_block(lap, poly, blk, a.d, out=out, work=work)
torch.cuda.synchronize()
print("ok", lap.nnz, lap.plan(1.0, dt).nnz)
