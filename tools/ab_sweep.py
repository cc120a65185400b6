"""Interleaved A/B of sweep tuning knobs inside one process (medians over rounds).

    python tools/ab_sweep.py --configs "chunk_bytes=512;chunk_bytes=1024" [--precision fp64] [--rounds 5]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import _native, generators as G  # noqa: E402
from paper_1706_03591_b200._device import row_stride  # noqa: E402
from paper_1706_03591_b200.filters import filter_block  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", required=True)
ap.add_argument("--precision", default="fp64")
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--orders", type=int, default=20)
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--workload", default="cfg3")
a = ap.parse_args()
if a.workload == "cfg4":
    n = 4_000_000
    g, _ = G.chung_lu_sbm(n, 50, 16.0, 2.3, 20000.0, 0.05, seed=4)
else:
    n, k, deg, ratio = {"cfg3": (1_000_000, 100, 32.0, 0.02), "cfg5": (2_000_000, 64, 20.0, 0.05),
                        "cfg2": (20_000, 20, 24.0, 0.05)}[a.workload]
    q1, q2 = G.sbm_probabilities(n, k, deg, ratio)
    g = G.graph_from_codes(n, G.planted_partition_codes(n, k, q1, q2, 3))
lap = P.laplacian(g)
dt = torch.float64 if a.precision == "fp64" else torch.float32
ld = row_stride(a.d, dt)
blk = torch.zeros((n, ld), dtype=dt, device="cuda")
blk[:, :a.d] = torch.randn((n, a.d), dtype=dt, device="cuda") / np.sqrt(a.d)
poly = P.cheb_coeffs(0.05, 2.0, a.orders)
out = torch.empty_like(blk)
work = torch.empty((2 * n, ld), dtype=dt, device="cuda")
configs = [dict(kv.split("=") for kv in c.split(",") if kv) for c in a.configs.split(";")]
lib = _native.lib()


def apply(cfg):
    for kk, vv in cfg.items():
        _native.check(lib.csc_set_tuning(kk.encode(), int(vv)), "tuning")


res = {i: [] for i in range(len(configs))}
for r in range(a.rounds):
    for i, cfg in enumerate(configs):
        apply(cfg)
        filter_block(lap, poly, blk, a.d, out=out, work=work)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        filter_block(lap, poly, blk, a.d, out=out, work=work)
        e1.record()
        torch.cuda.synchronize()
        res[i].append(e0.elapsed_time(e1) / a.orders)
nnz = lap.nnz
s = 8 if dt == torch.float64 else 4
bmin = 4 * (n + 1) + nnz * (4 + s) + nnz * a.d * s + n * a.d * s
for i, cfg in enumerate(configs):
    med = statistics.median(res[i])
    print(json.dumps({"cfg": cfg, "workload": a.workload, "precision": a.precision, "d": a.d,
                      "ms_per_order_median": round(med, 4), "min": round(min(res[i]), 4),
                      "max": round(max(res[i]), 4), "gbs_bmin": round(bmin / med / 1e6)}))
