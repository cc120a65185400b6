"""Program profiled by ncu for bench.py's `roofline.traffic` (tools only).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        -k regex:sweep_kernel --csv --log-file gpurun_out/traffic_<wl>_<prec>.csv \
        python tools/capture_traffic.py --workload cfg3 --precision fp64 > gpurun_out/traffic_<wl>_<prec>.json
    python tools/traffic_json.py gpurun_out/traffic_<wl>_<prec>   # -> profiles/r02_sweep_<wl>_<prec>.json

Builds the bench's graph and block, runs one order-4 filter (first + 3 middle
sweeps) and prints the kernel instance and grid of the last (middle) sweep —
the launch bench.py times — as one JSON line.
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import _native, generators as G  # noqa: E402
from paper_1706_03591_b200._device import row_stride  # noqa: E402
from paper_1706_03591_b200.filters import filter_block  # noqa: E402
from paper_1706_03591_b200.signals import device_signals  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg3", choices=["cfg3", "cfg4"])
ap.add_argument("--precision", default="fp64")
a = ap.parse_args()
if a.workload == "cfg3":
    w = bench.WORKLOADS["cfg3"]
    codes, _ = bench.make_graph_codes(w)
    g = G.graph_from_codes(w["n"], codes)
else:
    w = bench.CFG4
    cache = "/tmp/csc_cfg4_codes.npy"  # tool-side cache only
    if os.path.exists(cache):
        g = G.graph_from_codes(w["n"], np.load(cache))
    else:
        g, _ = G.chung_lu_sbm(w["n"], w["k"], w["deg"], w["exponent"], w["max_degree"], w["ratio"], seed=w["seed"])
        np.save(cache, g.edge_i * w["n"] + g.edge_j)
n, d = w["n"], w["d"]
lap = P.laplacian(g)
dt = torch.float64 if a.precision == "fp64" else torch.float32
plan = lap.plan(1.0, dt)
x = device_signals(n, d, 1)
blk = torch.zeros((n, row_stride(d, dt)), dtype=dt, device="cuda")
blk[:, :d].copy_(x[:, :d])
poly = P.cheb_coeffs(w["cutoff"], 2.0, 4)
filter_block(lap, poly, blk, d)
torch.cuda.synchronize()
name, grid = bench.last_launch(_native.lib())
s = 8 if dt == torch.float64 else 4
print(json.dumps({"workload": a.workload, "precision": a.precision, "kernel": name, "grid": grid,
                  "n": n, "nnz_L": int(lap.nnz), "d": d,
                  "bytes_min_per_launch": int(bench.b_min(n, lap.nnz, d, s))}))
