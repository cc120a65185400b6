"""Time the fused sweep on a synthetic workload: ms per order via CUDA events.

    python tools/time_sweep.py [--workload cfg3|cfg4|cfg5] [--precision fp64|fp32] [--d 128] [--orders 40]
"""
import argparse
import json
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
ap.add_argument("--orders", type=int, default=40)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--workload", default="cfg3")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
if a.workload == "cfg3":
    n, k, deg, ratio = 1_000_000, 100, 32.0, 0.02
elif a.workload == "cfg5":
    n, k, deg, ratio = 2_000_000, 64, 20.0, 0.05
if a.workload in ("cfg3", "cfg5"):
    q1, q2 = G.sbm_probabilities(n, k, deg, ratio)
    g = G.graph_from_codes(n, G.planted_partition_codes(n, k, q1, q2, 3))
else:
    n = 4_000_000
    g, _ = G.chung_lu_sbm_device(n, 50, 16.0, 2.3, 20000.0, 0.05, seed=4)
lap = P.laplacian(g)
dt = torch.float64 if a.precision == "fp64" else torch.float32
ld = row_stride(a.d, dt)
blk = torch.zeros((n, ld), dtype=dt, device="cuda")
blk[:, :a.d] = torch.randn((n, a.d), dtype=dt, device="cuda") / np.sqrt(a.d)
poly = P.cheb_coeffs(0.05, 2.0, a.orders)
out = torch.empty_like(blk)
work = torch.empty((2 * n, ld), dtype=dt, device="cuda")
filter_block(lap, poly, blk, a.d, out=out, work=work)
torch.cuda.synchronize()
best = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    filter_block(lap, poly, blk, a.d, out=out, work=work)
    e1.record()
    torch.cuda.synchronize()
    best.append(e0.elapsed_time(e1) / a.orders)
nnz = lap.nnz
s = 8 if dt == torch.float64 else 4
plan = lap.plan(1.0, dt)
bmin = 4 * (n + 1) + nnz * (4 + s) + nnz * a.d * s + n * a.d * s
ms = min(best)
print(json.dumps({"workload": a.workload, "precision": a.precision, "d": a.d, "n": n, "nnz_L": nnz,
                  "nnz_M": plan.nnz, "n_long": plan.n_long, "ms_per_order": ms, "all": best,
                  "units_per_s": nnz * a.d / (ms / 1e3), "gbs_bmin": bmin / (ms / 1e3) / 1e9,
                  "hint": os.environ.get("CSC_STREAM_HINT", "1")}))
