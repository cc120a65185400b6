"""A/B of the FP32 assignment screen on real CSC features (configs[4] shape by default).

Runs the lane-path k-means (run_restarts, fused=False) with the screen on and
off, interleaved; prints ms per call, iterations, and whether labels / cost
are identical.

    python tools/ab_screen.py [--n 2000000 --k 64 --d 96 --m 80 --restarts 2 --iters 30 --rounds 3]
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
from paper_1706_03591_b200._device import ptr  # noqa: E402
from paper_1706_03591_b200.filters import FilteredBlock, _search_cutoff  # noqa: E402
from paper_1706_03591_b200.signals import device_signals  # noqa: E402

KM = importlib.import_module("paper_1706_03591_b200.kmeans")
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2_000_000)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--d", type=int, default=96)
ap.add_argument("--m", type=int, default=80)
ap.add_argument("--deg", type=float, default=20.0)
ap.add_argument("--ratio", type=float, default=0.05)
ap.add_argument("--restarts", type=int, default=2)
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--rounds", type=int, default=3)
a = ap.parse_args()
q1, q2 = G.sbm_probabilities(a.n, a.k, a.deg, a.ratio)
g = G.graph_from_codes(a.n, G.planted_partition_codes(a.n, a.k, q1, q2, 5))
lap = P.laplacian(g)
blk = device_signals(a.n, a.d, 0)
cut, filt, poly, iters, est = _search_cutoff(lap, a.k, FilteredBlock(blk, a.d), (0.0, 2.0),
                                             P.FilterConfig(order=a.m), None, 1.0)
F = filt.blk
cfg = P.KmeansConfig(restarts=a.restarts, max_iters=a.iters)
kids = np.random.SeedSequence(1).spawn(a.restarts)
KM.run_restarts(F, a.d, a.k, cfg, kids, fused=False)  # warm: pool, graphs
pool = KM._LLOYD_POOL


def screen(on):
    for lane in pool.lanes:
        if on:
            _native.call("csc_kmeans_plan_set_screen", lane.plan, ptr(pool.F32), pool.ld32, ptr(pool.fn32))
        else:
            _native.call("csc_kmeans_plan_set_screen", lane.plan, None, 0, None)


res = {True: [], False: []}
out = {}
for r in range(a.rounds):
    for on in (True, False):
        screen(on)
        KM.run_restarts(F, a.d, a.k, cfg, kids, fused=False)  # graph rebuild outside the timing
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lab, cost = KM.run_restarts(F, a.d, a.k, cfg, kids, fused=False)
        torch.cuda.synchronize()
        res[on].append((time.perf_counter() - t0) * 1e3)
        out[on] = (lab, cost)
screen(True)
its = [int(pool.lanes[i].out[1].item()) for i in range(a.restarts)]
same = np.array_equal(out[True][0], out[False][0]) and out[True][1] == out[False][1]
print(f"n={a.n} d={a.d} k={a.k} restarts={a.restarts} iterations {its}: screen on "
      f"{np.median(res[True]):.1f} ms, off {np.median(res[False]):.1f} ms; identical labels+cost: {same}")
