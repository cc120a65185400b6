"""bench.py's configs[4] legs in bench order with per-step phase times and
memory state, to locate occasional slow steps (tools only).

    python tools/cfg5_hiccup_probe.py [--warm-cfg3]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import generators as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--warm-cfg3", action="store_true")
ap.add_argument("--sync", action="store_true", help="synchronise at every phase mark")
ap.add_argument("--nosync-marks", action="store_true")
ap.add_argument("--fine", action="store_true", help="synchronised timers around apply_delta / laplacian / plan")
a = ap.parse_args()

import importlib  # noqa: E402
D = importlib.import_module("paper_1706_03591_b200.dynamic")
orig_step = P.dynamic_step
if a.sync:
    real = D.time.perf_counter

    def synced():
        torch.cuda.synchronize()
        return real()

    class _T:
        perf_counter = staticmethod(synced)

    D.time = _T


def step(state, g, cfg, timings=None, **kw):
    ph = {}
    t0 = time.perf_counter()
    out = orig_step(state, g, cfg, timings=ph, **kw)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    free, total = torch.cuda.mem_get_info()
    import numpy as _np
    from paper_1706_03591_b200 import _native as _nv
    st = _np.zeros(4, dtype=_np.int64)
    _nv.call("csc_pool_stats", st.ctypes.data)
    print("  pool reserved %.2f used %.2f high %.2f / %.2f GiB" % tuple(st / 2**30), flush=True)
    print(f"  step {ms:7.1f} ms  " + " ".join(f"{k}={v:.1f}" for k, v in ph.items())
          + f" | free {free / 2**30:.1f} GiB torch reserved {torch.cuda.memory_reserved() / 2**30:.1f}", flush=True)
    if timings is not None:
        for k, v in ph.items():
            timings[k] = timings.get(k, 0.0) + v
    return out


P.dynamic_step = step

# finer marks inside the first phase (each synchronised)
GR = importlib.import_module("paper_1706_03591_b200.graphs")


def timed(name, fn):
    def w(*x, **kw):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*x, **kw)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        if ms > 30.0:
            print(f"    slow {name}: {ms:.1f} ms", flush=True)
        return r
    return w


def timed_nosync(name, fn):
    def w(*x, **kw):
        t0 = time.perf_counter()
        r = fn(*x, **kw)
        ms = (time.perf_counter() - t0) * 1e3
        if ms > 30.0:
            print(f"    slow (no sync) {name}: {ms:.1f} ms", flush=True)
        return r
    return w


if a.nosync_marks:
    from paper_1706_03591_b200 import _native as NV
    real_call = NV.call

    def call(name, *x):
        t0 = time.perf_counter()
        r = real_call(name, *x)
        ms = (time.perf_counter() - t0) * 1e3
        if ms > 30.0 and name in ("csc_laplacian_build", "csc_edge_delta", "csc_chebop_create", "csc_chebop_destroy"):
            print(f"    slow native {name}: {ms:.1f} ms", flush=True)
        return r

    NV.call = call
    GR._native.call = call
    D.laplacian = timed_nosync("laplacian()", D.laplacian)
    GR.LaplacianMatrix.plan = timed_nosync("plan()", GR.LaplacianMatrix.plan)
    GR.Graph.apply_delta = timed_nosync("apply_delta()", GR.Graph.apply_delta)
    GR.Graph.device_edges = timed_nosync("device_edges()", GR.Graph.device_edges)
    real_empty = torch.empty

    def empty(*x, **kw):
        t0 = time.perf_counter()
        r = real_empty(*x, **kw)
        ms = (time.perf_counter() - t0) * 1e3
        if ms > 30.0:
            print(f"    slow torch.empty{x}: {ms:.1f} ms", flush=True)
        return r

    GR.torch.empty = empty
if a.fine:
    D.laplacian = timed("laplacian()", D.laplacian)
    GR.LaplacianMatrix.plan = timed("plan()", GR.LaplacianMatrix.plan)
    GR.Graph.apply_delta = timed("apply_delta()", GR.Graph.apply_delta)
    GR.Graph.device_edges = timed("device_edges()", GR.Graph.device_edges)
if a.warm_cfg3:
    wc = bench.WORKLOADS["cfg3"]
    codes3, _ = bench.make_graph_codes(wc)
    lap3 = P.laplacian(G.graph_from_codes(wc["n"], codes3))
    print(bench.run_cfg3_pipeline(lap3, wc), flush=True)
    del lap3
    torch.cuda.empty_cache()


class A:
    pass


print("dynamic_cfg5", flush=True)
r = bench.run_dynamic_cfg5(A(), 0)
print(r["ms_all"], flush=True)
print("matrix", flush=True)
m = bench.run_dynamic_cfg5_matrix(0)
for c in m["cells"] + m["quality"]["cells"]:
    print(c["churn"], c["p"], c["ms_all"], flush=True)
