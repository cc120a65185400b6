"""k-means plan modes at the cfg3 shape against the oracle (tools only): the
tensor-core / SIMT / FP64-only assignment screens with and without the
incremental centroid sums, each run from the same seed as the oracle's
k-means++ + Lloyd (kmeans.py:64-117).

    python tools/debug_kmeans_modes.py [--n 1000000] [--iters 3]
"""
import argparse
import importlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import _native  # noqa: E402
from paper_1706_03591_b200 import generators as G  # noqa: E402
from paper_1706_03591_b200.filters import filter_block  # noqa: E402
from paper_1706_03591_b200.signals import device_signals  # noqa: E402
from oracle import csc_oracle as O  # noqa: E402

KM = importlib.import_module("paper_1706_03591_b200.kmeans")
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--k", type=int, default=100)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--restarts", type=int, default=1)
ap.add_argument("--no-oracle", action="store_true")
a = ap.parse_args()
n, k, d = a.n, a.k, a.d
q1, q2 = G.sbm_probabilities(n, k, 32.0, 0.02)
g = G.graph_from_codes(n, G.planted_partition_codes(n, k, q1, q2, 3))
lap = P.laplacian(g)
x = device_signals(n, d, 30)
poly = P.cheb_coeffs(0.05, lap.lambda_max_bound, 40)
feats, _ = filter_block(lap, poly, x, d)
F = feats[:, :d]
cfg = P.KmeansConfig(restarts=a.restarts, max_iters=a.iters)
if not a.no_oracle:
    t0 = time.time()
    fh = F.cpu().numpy()
    ref_labels, _, ref_cost = O.kmeans(fh, k, restarts=a.restarts, max_iters=a.iters, seed=8)
    print(f"oracle {time.time() - t0:.1f} s cost {ref_cost:.12g}", flush=True)
res = {}
for name, tc, inc, screen in [("tc+inc", 1, 1, True), ("tc", 1, 0, True), ("simt+inc", 0, 1, True),
                              ("simt", 0, 0, True), ("fp64+inc", 0, 1, False), ("fp64", 0, 0, False)]:
    _native.call("csc_kmeans_tuning", b"screen_tc", tc)
    _native.call("csc_kmeans_tuning", b"update_incremental", inc)
    P.kmeans(F, k, cfg, seed=8)  # builds the pool
    pool = KM._LLOYD_POOL
    for lane in pool.lanes:
        if screen:
            _native.call("csc_kmeans_plan_set_screen", lane.plan, KM.ptr(pool.F32), pool.ld32, KM.ptr(pool.fn32))
        else:
            _native.call("csc_kmeans_plan_set_screen", lane.plan, None, 0, None)
    r = P.kmeans(F, k, cfg, seed=8)
    res[name] = r
    line = f"{name:9s} cost {r.feature_cost:.12g}"
    if not a.no_oracle:
        line += f" ARI {O.adjusted_rand(r.labels, ref_labels):.6f} rel {abs(r.feature_cost - ref_cost) / ref_cost:.2e}"
    line += f" == fp64: {np.array_equal(r.labels, res.get('fp64', r).labels)}"
    print(line, flush=True)
base = res["fp64"]
for name, r in res.items():
    diff = np.flatnonzero(r.labels != base.labels)
    print(f"{name:9s} vs fp64: {diff.size} labels differ, first {diff[:8]}")
