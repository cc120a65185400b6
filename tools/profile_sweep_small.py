"""cfg2-size sweeps (n=20k, d=40 fresh columns, order 60) for ncu / timing."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import generators as G  # noqa: E402
from paper_1706_03591_b200.filters import filter_block  # noqa: E402
from paper_1706_03591_b200.signals import device_signals  # noqa: E402

n, k, d = 20000, 20, int(sys.argv[1]) if len(sys.argv) > 1 else 40
q1, q2 = G.sbm_probabilities(n, k, 24.0, 0.05)
lap = P.laplacian(G.graph_from_codes(n, G.planted_partition_codes(n, k, q1, q2, 7)))
x = device_signals(n, d, 0)
poly = P.cheb_coeffs(0.3, lap.lambda_max_bound, 60)
out = torch.empty_like(x)
work = torch.empty((2 * n, x.shape[1]), dtype=x.dtype, device=x.device)
for _ in range(3):
    filter_block(lap, poly, x, d, out=out, work=work)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    filter_block(lap, poly, x, d, out=out, work=work)
torch.cuda.synchronize()
ms = (time.perf_counter() - t0) / 10 * 1e3
print(f"n={n} d={d} nnz={lap.nnz}: {ms:.3f} ms per 60-order filter = {ms / 60 * 1e3:.1f} us/order")
