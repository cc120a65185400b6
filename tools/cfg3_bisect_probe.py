"""Where the time of a configs[2] lambda_k search goes (tools only): synchronised
timers around the resident-orders allocation, the moment pass, the exact
combinations and any fallback sweep series.

    python tools/cfg3_bisect_probe.py [--calls 4]
"""
import argparse
import importlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import generators as G  # noqa: E402
from paper_1706_03591_b200.signals import device_signals  # noqa: E402

F = importlib.import_module("paper_1706_03591_b200.filters")
ap = argparse.ArgumentParser()
ap.add_argument("--calls", type=int, default=4)
ap.add_argument("--kmeans", action="store_true", help="run the k-means of csc_assign after each search")
a = ap.parse_args()
w = bench.WORKLOADS["cfg3"]
codes, _ = bench.make_graph_codes(w)
lap = P.laplacian(G.graph_from_codes(w["n"], codes))
k, d = w["k"], w["d"]
cfg = P.FilterConfig(order=w["order"])
log = []


def timed(name):
    fn = getattr(F, name)

    def wrap(*x, **kw):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*x, **kw)
        torch.cuda.synchronize()
        log.append((name, (time.perf_counter() - t0) * 1e3))
        return r

    setattr(F, name, wrap)


for nm in ("resident_orders", "block_moments_keep", "block_moments", "combine_orders", "filter_block"):
    timed(nm)
for c in range(a.calls):
    blk = device_signals(lap.n, d, np.random.SeedSequence(c).spawn(2)[0])
    torch.cuda.synchronize()
    log.clear()
    t0 = time.perf_counter()
    out = F._search_cutoff(lap, k, F.FilteredBlock(blk, d), (0.0, lap.lambda_max_bound), cfg, None, 1.0)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    free, total = torch.cuda.mem_get_info()
    print(f"call {c}: {ms:.1f} ms, {out[3]} probes; " + ", ".join(f"{n} {t:.1f}" for n, t in log)
          + f" | free {free / 2**30:.1f} GiB, torch reserved {torch.cuda.memory_reserved() / 2**30:.1f}", flush=True)
    if a.kmeans:
        KM = importlib.import_module("paper_1706_03591_b200.kmeans")
        kids = np.random.SeedSequence(c).spawn(2)[1].spawn(10)
        t0 = time.perf_counter()
        KM.run_restarts(out[1].blk, d, k, P.KmeansConfig(), kids)
        torch.cuda.synchronize()
        print(f"   k-means {(time.perf_counter() - t0) * 1e3:.1f} ms; torch reserved {torch.cuda.memory_reserved() / 2**30:.1f} "
              f"allocated {torch.cuda.memory_allocated() / 2**30:.1f} GiB", flush=True)
    del out
