"""Would an fp32 GEMM-form screen decide k-means labels on real CSC features?

Exact fp64 Lloyd in torch on cfg5-shape features; per iteration, the
fraction of rows whose fp32 best/second gap exceeds the rigorous bound
2 (d+4) u32 (|f| + max|c|)^2 (those rows' fp64 argmin is provably the fp32
one), and the actual max |E32 - D64| relative to that bound.

    python tools/fp32_screen_sim.py [--n 2000000 --k 64 --d 96 --m 80 --iters 30]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import generators as G  # noqa: E402
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
ap.add_argument("--iters", type=int, default=30)
a = ap.parse_args()
q1, q2 = G.sbm_probabilities(a.n, a.k, a.deg, a.ratio)
g = G.graph_from_codes(a.n, G.planted_partition_codes(a.n, a.k, q1, q2, 5))
lap = P.laplacian(g)
blk = device_signals(a.n, a.d, 0)
cut, filt, poly, iters, est = _search_cutoff(lap, a.k, FilteredBlock(blk, a.d), (0.0, 2.0),
                                             P.FilterConfig(order=a.m), None, 1.0)
ws = _Workspace(filt.blk, a.d, a.k)
seeds = batched_kmeanspp(ws, np.random.SeedSequence(1).spawn(1))
F = filt.blk[:, :a.d].contiguous()
C = seeds[0][:, :a.d].clone()
F32 = F.float()
fn = (F * F).sum(1)
fnorm = fn.sqrt()
u32 = 2.0 ** -24
for it in range(a.iters):
    cn = (C * C).sum(1)
    D = (fn[:, None] - 2.0 * (F @ C.T)) + cn[None, :]
    D.clamp_(min=0.0)
    C32 = C.float()
    E = ((F32 * F32).sum(1)[:, None] - 2.0 * (F32 @ C32.T)) + (C32 * C32).sum(1)[None, :]
    E = E.double()
    bound = (a.d + 4) * u32 * (fnorm + cn.sqrt().max()) ** 2
    err = (E - D).abs().max(1).values
    top2 = E.topk(2, dim=1, largest=False).values
    gap = top2[:, 1] - top2[:, 0]
    decided = (gap > 2.0 * bound).float().mean().item()
    lab = D.argmin(1)
    lab32 = E.argmin(1)
    wrong_decided = ((lab != lab32) & (gap > 2.0 * bound)).sum().item()
    print(f"it {it:3d}: decided {100 * decided:6.2f}%  max err/bound {(err / bound).max().item():.3f}  "
          f"median gap/bound {(gap / bound).median().item():.1f}  wrong-but-decided {wrong_decided}", flush=True)
    sums = torch.zeros_like(C).index_add_(0, lab, F)
    cnt = torch.bincount(lab, minlength=a.k).clamp(min=1)
    C = sums / cnt[:, None].double()
