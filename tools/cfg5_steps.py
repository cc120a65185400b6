"""Per-phase times of configs[4] dynamic steps (tools only): like bench.py's
dynamic_cfg5 but with a device synchronisation at every phase mark, so the
phase split is exact; also the k-means restarts' iteration counts.

    python tools/cfg5_steps.py [--steps 4] [--p 0.5] [--churn 0.01]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import generators as G  # noqa: E402
import importlib  # noqa: E402

K = importlib.import_module("paper_1706_03591_b200.kmeans")
D = importlib.import_module("paper_1706_03591_b200.dynamic")
ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--p", type=float, default=0.5)
ap.add_argument("--churn", type=float, default=0.01)
ap.add_argument("--warm-cfg3", action="store_true", help="run the cfg3 csc_assign pipeline first (bench order)")
a = ap.parse_args()
if a.warm_cfg3:
    wc = bench.WORKLOADS["cfg3"]
    codes3, _ = bench.make_graph_codes(wc)
    lap3 = P.laplacian(G.graph_from_codes(wc["n"], codes3))
    for s3 in range(3):
        t0 = time.perf_counter()
        P.csc_assign(lap3, wc["k"], wc["d"], P.FilterConfig(order=wc["order"]), P.KmeansConfig(), seed=s3)
        torch.cuda.synchronize()
        print(f"cfg3 csc_assign {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
    del lap3
w = bench.WORKLOADS["cfg5"]
n, k, d = w["n"], w["k"], w["d"]
q1, q2 = G.sbm_probabilities(n, k, w["deg"], w["ratio"])
g, labels = G.planted_partition_device(n, k, w["deg"], w["ratio"], seed=w["seed"])
deltas, cur = [], g
for s in range(a.steps):
    dl, il = G.edge_churn_device(cur, labels, q1, q2, a.churn, seed=50 + s)
    cur = cur.apply_delta(dl, il)
    deltas.append((dl.cpu().numpy(), il.cpu().numpy()))
cfg = P.DynamicConfig(k=k, d=d, p=a.p, filter=P.FilterConfig(order=w["order"]))
torch.cuda.synchronize()
t0 = time.perf_counter()
_, state, diag0 = P.dynamic_init(g, cfg, seed=0)
torch.cuda.synchronize()
print(f"init {(time.perf_counter() - t0) * 1e3:.1f} ms, search iters {diag0.search_iters}", flush=True)
orig_time = D.time.perf_counter


def synced():
    torch.cuda.synchronize()
    return orig_time()


D.time.perf_counter = synced  # phase marks after a device sync (tools only)
for dl, il in deltas:
    ph = {}
    torch.cuda.synchronize()
    t0 = orig_time()
    g = g.apply_delta(dl, il)
    torch.cuda.synchronize()
    t1 = orig_time()
    asg, state, diag = P.dynamic_step(state, g, cfg, timings=ph)
    torch.cuda.synchronize()
    t2 = orig_time()
    pool = K._LLOYD_POOL
    its = [int(pool.lanes[i].out[1].item()) for i in range(cfg.kmeans.restarts)] if pool else []
    print(f"[replays {K.KPP_REPLAYS[0]}] ", end="")
    print(f"step {(t2 - t0) * 1e3:.1f} ms: delta {(t1 - t0) * 1e3:.1f} "
          + " ".join(f"{kk} {v:.1f}" for kk, v in ph.items())
          + f" | refined {diag.refined} | kmeans iters {its}", flush=True)
