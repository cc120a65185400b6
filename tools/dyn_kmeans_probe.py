"""configs[1] dynamic sequence: per-step k-means time, seeding time and Lloyd iterations per restart.

Same graph sequence as bench.run_dynamic; prints one line per step.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import generators as G  # noqa: E402
import importlib  # noqa: E402
KM = importlib.import_module("paper_1706_03591_b200.kmeans")


def sequence(steps=10):
    n, k = 20000, 20
    q1, q2 = G.sbm_probabilities(n, k, 24.0, 0.05)
    codes = G.planted_partition_codes(n, k, q1, q2, 7)
    labels = np.repeat(np.arange(k), G.block_sizes(n, k))
    graphs = [G.graph_from_codes(n, codes)]
    cur = codes

    def applied(c, dl, il):
        return np.union1d(np.setdiff1d(c, dl, assume_unique=True), il)

    for t in range(1, steps):
        dn, inn, labels = G.node_switch(cur, n, labels, k, q1, q2, 0.005, seed=200 + t)
        cur = applied(cur, dn, inn)
        de, ie = G.edge_churn(cur, n, labels, q1, q2, 0.01, seed=100 + t)
        graphs.append(graphs[-1].apply_delta(dn, inn).apply_delta(de, ie))
        cur = applied(cur, de, ie)
    return graphs


def main():
    graphs = sequence()
    cfg = P.DynamicConfig(k=20, d=80, p=0.5, filter=P.FilterConfig(order=60))
    thetas = []
    orig = KM._kmeans_prepared

    def spy(theta, d, k, kcfg, children, draws):
        thetas.append((theta.clone(), children, draws))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a = orig(theta, d, k, kcfg, children, draws)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        pool = KM._LLOYD_POOL
        if os.environ.get("CSC_KMEANS_FUSED", "1") != "0":
            its = list(KM.LAST_FUSED_ITERS)
        else:
            its = [int(pool.lanes[i].out[1].item()) for i in range(kcfg.restarts)]
        print(f"kmeans {ms:.2f} ms iterations {its} sum {sum(its)}", flush=True)
        return a

    D = importlib.import_module("paper_1706_03591_b200.dynamic")
    D._kmeans_prepared = spy
    for rep in range(2):
        print(f"--- pass {rep}")
        _, state, _ = P.dynamic_init(graphs[0], cfg, seed=0)
        for gt in graphs[1:]:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ph = {}
            _, state, _ = P.dynamic_step(state, gt, cfg, timings=ph)
            torch.cuda.synchronize()
            print(f"step {(time.perf_counter() - t0) * 1e3:.2f} ms " +
                  " ".join(f"{a}={b:.2f}" for a, b in ph.items()), flush=True)
    if os.environ.get("SAVE_THETA"):
        th, children, draws = thetas[-1]
        np.save(os.environ["SAVE_THETA"], th[:, :80].cpu().numpy())


if __name__ == "__main__":
    main()
