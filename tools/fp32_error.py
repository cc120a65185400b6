"""fp32 filter error vs fp64 (cfg1 vs the reference golden; cfg3 vs the fp64 GPU result)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import generators as G  # noqa: E402
from paper_1706_03591_b200.filters import filter_block  # noqa: E402
from paper_1706_03591_b200.signals import device_signals  # noqa: E402

res = {}
g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "cfg1.npz"))
lap = P.laplacian(P.Graph(1000, g["g_i"], g["g_j"], g["g_w"]))
poly = P.cheb_coeffs(0.5, 2.0, 50)
o32 = P.apply_filter(lap, poly, g["R"], precision="fp32")
res["cfg1_m50_fp32_rel_frobenius_vs_reference"] = float(np.linalg.norm(o32 - g["filt_05"]) / np.linalg.norm(g["filt_05"]))
n, k = 1_000_000, 100
q1, q2 = G.sbm_probabilities(n, k, 32.0, 0.02)
lap3 = P.laplacian(G.graph_from_codes(n, G.planted_partition_codes(n, k, q1, q2, 3)))
blk = device_signals(n, 128, 0)
for cut in (0.05, 0.6):
    p = P.cheb_coeffs(cut, 2.0, 100)
    o64, s64 = filter_block(lap3, p, blk, 128, want_sumsq=True)
    o32, s32 = filter_block(lap3, p, blk.to(torch.float32), 128, want_sumsq=True)
    diff = (o64 - o32.to(torch.float64)).norm() / o64.norm()
    res[f"cfg3_m100_cut{cut}_fp32_rel_frobenius_vs_fp64"] = float(diff)
    res[f"cfg3_m100_cut{cut}_eigencount_fp64_fp32"] = [float(s64.item()), float(s32.item())]
print(json.dumps(res))
