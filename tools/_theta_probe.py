import os, sys, time, importlib
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import numpy as np, torch
import paper_1706_03591_b200 as P
from dyn_kmeans_probe import sequence
S = importlib.import_module("paper_1706_03591_b200.signals")
D = importlib.import_module("paper_1706_03591_b200.dynamic")
graphs = sequence(6)
cfg = P.DynamicConfig(k=20, d=80, p=0.5, filter=P.FilterConfig(order=60))
T = {}
def timed(name, fn):
    def w(*a, **k):
        t0 = time.perf_counter(); r = fn(*a, **k); T[name] = T.get(name, 0) + (time.perf_counter() - t0) * 1e3; return r
    return w
D.gather_columns = timed("gather", S.gather_columns)
orig_fb = S.FeatureMatrix._from_block.__func__
S.FeatureMatrix._from_block = classmethod(timed("from_block", orig_fb))
D.FeatureMatrix = S.FeatureMatrix
ozeros = torch.zeros
D.torch = type("T", (), {})()
for nm in dir(torch):
    try: setattr(D.torch, nm, getattr(torch, nm))
    except Exception: pass
D.torch.zeros = timed("zeros", ozeros)
_, state, _ = P.dynamic_init(graphs[0], cfg, seed=0)
for gt in graphs[1:]:
    ph = {}
    T.clear()
    torch.cuda.synchronize()
    _, state, _ = P.dynamic_step(state, gt, cfg, timings=ph)
    print({k: round(v, 3) for k, v in ph.items()}, {k: round(v, 3) for k, v in T.items()})
