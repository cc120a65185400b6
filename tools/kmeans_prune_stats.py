"""Pruning effectiveness of the bounds-pruned Lloyd plan on real CSC features.

Builds a planted-partition graph, filters signals at a cutoff found by the
moment bisection, then runs one restart of Lloyd recording per-iteration
candidates and times.   python tools/kmeans_prune_stats.py [--n 2000000 --k 64 --d 96 --m 80]
"""
import argparse
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import _native, generators as G  # noqa: E402
from paper_1706_03591_b200._device import ptr, stream  # noqa: E402
from paper_1706_03591_b200.filters import FilteredBlock, _search_cutoff  # noqa: E402
from paper_1706_03591_b200.kmeans import _Workspace, batched_kmeanspp  # noqa: E402
from paper_1706_03591_b200.signals import device_signals  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2_000_000)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--d", type=int, default=96)
ap.add_argument("--m", type=int, default=80)
ap.add_argument("--deg", type=float, default=20.0)
ap.add_argument("--ratio", type=float, default=0.05)
ap.add_argument("--iters", type=int, default=100)
a = ap.parse_args()
q1, q2 = G.sbm_probabilities(a.n, a.k, a.deg, a.ratio)
g = G.graph_from_codes(a.n, G.planted_partition_codes(a.n, a.k, q1, q2, 5))
lap = P.laplacian(g)
blk = device_signals(a.n, a.d, 0)
cut, filt, poly, iters, est = _search_cutoff(lap, a.k, FilteredBlock(blk, a.d), (0.0, 2.0),
                                             P.FilterConfig(order=a.m), None, 1.0)
ws = _Workspace(filt.blk, a.d, a.k)
seeds = batched_kmeanspp(ws, np.random.SeedSequence(1).spawn(1))
ws.cent.copy_(seeds[0])
plan = ws._plan()
s = stream()
_native.call("csc_kmeans_rownorms", ptr(ws.cent), a.k, a.d, ws.ldc, ptr(ws.cnorm), s)
rows = []
prev = np.inf
for it in range(a.iters):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _native.call("csc_kmeans_iterate", plan, ptr(ws.blk), ptr(ws.fnorm), ptr(ws.cent), ws.ldc, ptr(ws.cnorm),
                 ptr(ws.labels), ptr(ws.counts), int(it == 0), ptr(ws.scalars[1:]), s)
    cost2 = float(ws.scalars[1].item())
    ms = (time.perf_counter() - t0) * 1e3
    cand = ctypes.c_int64(0)
    gated = ctypes.c_int32(0)
    _native.call("csc_kmeans_plan_stats", plan, ctypes.byref(cand), ctypes.byref(gated))
    rows.append((it, round(ms, 3), int(cand.value) if it else a.n, int(gated.value), cost2))
    stop = np.isfinite(prev) and prev - cost2 <= 1e-6 * prev
    prev = cost2
    if stop:
        break
tot = sum(r[1] for r in rows)
print(json.dumps({"total_ms": round(tot, 1), "cutoff": cut, "probe_iters": iters, "est": est, "iterations": len(rows),
                  "per_iter": rows[:5] + rows[5::10] + rows[-3:]}))
