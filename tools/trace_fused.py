"""Phase timeline of the fused Lloyd launch (csc_kmeans_fused_trace) on a configs[1] Theta.

Runs the configs[1] dynamic sequence to step 3 (the same Theta as the bench),
then one fused k-means of that Theta with CTA 0's globaltimer recorded at each
phase boundary; prints per-iteration phase durations (us).
"""
import importlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import _native  # noqa: E402
from paper_1706_03591_b200._device import ptr  # noqa: E402

KM = importlib.import_module("paper_1706_03591_b200.kmeans")
D = importlib.import_module("paper_1706_03591_b200.dynamic")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from dyn_kmeans_probe import sequence  # noqa: E402

graphs = sequence(4)
cfg = P.DynamicConfig(k=20, d=80, p=0.5, filter=P.FilterConfig(order=60))
captured = []
orig = KM._kmeans_prepared


def spy(theta, d, k, kcfg, children, draws):
    captured.append((theta.clone(), children, draws))
    return orig(theta, d, k, kcfg, children, draws)


D._kmeans_prepared = spy
_, state, _ = P.dynamic_init(graphs[0], cfg, seed=0)
for gt in graphs[1:]:
    _, state, _ = P.dynamic_step(state, gt, cfg)
cap = 128
trace = torch.zeros(cap * 16, dtype=torch.int64, device="cuda")
for which in range(len(captured)):
    theta, children, draws = captured[which]
    for rep in range(2):
        _native.call("csc_kmeans_fused_trace", ptr(trace), cap)
        trace.zero_()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        KM.run_restarts(theta, 80, 20, cfg.kmeans, children, draws, fused=True)
        ev1.record()
        torch.cuda.synchronize()
        _native.call("csc_kmeans_fused_trace", None, 0)
    t = trace.cpu().numpy().reshape(cap, 16).astype(np.float64)
    its = KM.LAST_FUSED_ITERS
    G = max(its) + 1
    t = t[:G]
    print(f"Theta {which}: kmeans call {ev0.elapsed_time(ev1):.3f} ms, iterations {its}, "
          f"kernel {(t[-1, 5] - t[0, 0]) / 1e3:.1f} us")
    names = ["phase1", "bar1", "phase2", "bar2", "tail"]
    for g in range(G):
        row = [(t[g, s + 1] - t[g, s]) / 1e3 for s in range(5)]
        act = sum(1 for v in its if v >= g)
        sub = [(t[g, 6] - t[g, 0]) / 1e3, (t[g, 7] - t[g, 6]) / 1e3, (t[g, 8] - t[g, 7]) / 1e3,
               (t[g, 9] - t[g, 8]) / 1e3, (t[g, 10] - t[g, 9]) / 1e3]
        print(f"  g={g:3d} active={act:2d} " + " ".join(f"{n}={v:7.1f}" for n, v in zip(names, row))
              + "  [first restart: load %.1f cost %.1f bounds %.1f assign %.1f (%d rows) sums %.1f]"
              % (sub[0], sub[1], sub[2], sub[3], int(t[g, 11]), sub[4]))
    kp = t_all = trace.cpu().numpy().reshape(cap, 16).astype(np.float64)[96:96 + 32]
    for j in range(32):
        if kp[j, 0] == 0:
            break
        print("  kpp draw %2d: dist+prefix %.1f  bar1 %.1f  draw %.1f  bar2 %.1f  stage %.1f" % (
            j, (kp[j, 1] - kp[j, 0]) / 1e3, 0.0, (kp[j, 2] - kp[j, 1]) / 1e3, (kp[j, 3] - kp[j, 2]) / 1e3,
            (kp[j, 4] - kp[j, 3]) / 1e3))
