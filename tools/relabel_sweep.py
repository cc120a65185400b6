"""Sweep roofline under node relabelling (tools only): cfg3 as generated
(block-contiguous node ids), randomly relabelled, and relabelled then
reordered by reverse Cuthill-McKee (scipy, host; an upper bound for what a
locality-restoring permutation buys). ms per order by CUDA events, B_min
fraction of the measured copy bandwidth.

    python tools/relabel_sweep.py [--precision fp64] [--orders 20]
"""
import argparse
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

ap = argparse.ArgumentParser()
ap.add_argument("--precision", default="fp64")
ap.add_argument("--orders", type=int, default=20)
a = ap.parse_args()
w = bench.WORKLOADS["cfg3"]
n, d = w["n"], w["d"]
codes, _ = bench.make_graph_codes(w)
lo, hi = codes // n, codes % n
perm = np.random.default_rng(17).permutation(n)


def relabel(mapping):
    i, j = mapping[lo], mapping[hi]
    c = np.minimum(i, j) * n + np.maximum(i, j)
    c.sort()
    return c


hbm, _ = bench.peaks()
dt = torch.float64 if a.precision == "fp64" else torch.float32
lib = _native.lib()
out = {}
cases = {"generated": codes, "random_relabel": relabel(perm)}
try:
    import scipy.sparse as sp
    from scipy.sparse.csgraph import reverse_cuthill_mckee
    rc = relabel(perm)
    A = sp.csr_matrix((np.ones(rc.size), (rc // n, rc % n)), shape=(n, n))
    A = A + A.T
    order = reverse_cuthill_mckee(A.tocsr(), symmetric_mode=True)
    inv = np.empty(n, np.int64)
    inv[order] = np.arange(n)
    cases["random_then_rcm"] = np.sort(np.minimum(inv[rc // n], inv[rc % n]) * n + np.maximum(inv[rc // n], inv[rc % n]))
except Exception as exc:  # noqa: BLE001
    out["rcm_error"] = str(exc)
for name, c in cases.items():
    lap = P.laplacian(G.graph_from_codes(n, c))
    blk = torch.zeros((n, row_stride(d, dt)), dtype=dt, device="cuda")
    blk[:, :d] = torch.randn((n, d), dtype=dt, device="cuda") / np.sqrt(d)
    outb = torch.empty_like(blk)
    work = torch.empty((2 * n, blk.shape[1]), dtype=dt, device="cuda")
    poly = P.cheb_coeffs(0.05, 2.0, a.orders)
    ms, sw = bench.timed_filter(lap, poly, blk, d, outb, work, 2, lib)
    s = 8 if dt == torch.float64 else 4
    bm = bench.b_min(n, lap.nnz, d, s)
    out[name] = {"sweep_ms": float(sw.mean()), "frac_bmin": bm / (float(sw.mean()) / 1e3) / 1e9 / hbm,
                 "schedule": "length_order" if lap.plan(1.0, dt).binned else "index_order"}
    print(name, json.dumps(out[name]), flush=True)
    del lap, blk, outb, work
    torch.cuda.empty_cache()
print(json.dumps(out))
