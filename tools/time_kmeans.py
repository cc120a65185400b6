"""k-means at scale on synthetic blob features: per-phase timing.

    python tools/time_kmeans.py [--n 2000000 --d 96 --k 64 --restarts 2 --iters 20]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200._device import row_stride  # noqa: E402
from paper_1706_03591_b200.kmeans import _Workspace  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2_000_000)
ap.add_argument("--d", type=int, default=96)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--restarts", type=int, default=2)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--tn", type=int, default=0)
ap.add_argument("--unpruned", action="store_true")
ap.add_argument("--ver", type=int, default=0)
a = ap.parse_args()
if a.tn:
    from paper_1706_03591_b200 import _native
    _native.check(_native.lib().csc_kmeans_tuning(b"assign_tn", a.tn), "tuning")
if a.ver:
    from paper_1706_03591_b200 import _native
    _native.check(_native.lib().csc_kmeans_tuning(b"assign_ver", a.ver), "tuning")
g = torch.Generator(device="cuda").manual_seed(0)
centers = torch.randn((a.k, a.d), dtype=torch.float64, device="cuda", generator=g) * 0.05
lab = torch.randint(0, a.k, (a.n,), device="cuda", generator=g)
blk = torch.zeros((a.n, row_stride(a.d)), dtype=torch.float64, device="cuda")
blk[:, :a.d] = centers[lab] + torch.randn((a.n, a.d), dtype=torch.float64, device="cuda", generator=g) * 0.02
ws = _Workspace(blk, a.d, a.k)
res = {}
for r in range(a.restarts):
    rng = np.random.default_rng(r)
    torch.cuda.synchronize(); t = time.perf_counter()
    ws.kmeanspp(rng)
    torch.cuda.synchronize(); res.setdefault("kmeanspp_ms", []).append((time.perf_counter() - t) * 1e3)
    hist = []
    t = time.perf_counter()
    ws.lloyd(a.iters, 0.0, hist, pruned=not a.unpruned)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) * 1e3
    res.setdefault("lloyd_ms_per_iter", []).append(dt / len(hist))
    res.setdefault("final_cost", []).append(float(hist[-1]))
print(json.dumps({"n": a.n, "d": a.d, "k": a.k, **res}))
