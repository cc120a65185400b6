"""Hamerly candidates with and without upper-bound tightening on real cfg5
features (tools only). Exact Lloyd in torch fp64; the bounds are tracked the
way the device plan keeps them (candidates get exact ub / lb from the full
evaluation, the other rows propagate ub += delta_a, lb -= max delta), and a
second copy tightens ub to the exact own distance before declaring a row a
candidate (one distance instead of k).

    python tools/hamerly_tight_sim.py [--iters 100]
"""
import argparse
import json
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
ap.add_argument("--iters", type=int, default=100)
a = ap.parse_args()
q1, q2 = G.sbm_probabilities(a.n, a.k, 20.0, 0.05)
g = G.graph_from_codes(a.n, G.planted_partition_codes(a.n, a.k, q1, q2, 5))
lap = P.laplacian(g)
blk = device_signals(a.n, a.d, 0)
cut, filt, poly, iters, est = _search_cutoff(lap, a.k, FilteredBlock(blk, a.d), (0.0, 2.0),
                                             P.FilterConfig(order=a.m), None, 1.0)
ws = _Workspace(filt.blk, a.d, a.k)
seeds = batched_kmeanspp(ws, np.random.SeedSequence(1).spawn(1))
F = filt.blk[:, :a.d].contiguous()
C = seeds[0][:, :a.d].clone()
n, k = a.n, a.k
ar = torch.arange(n, device=F.device)


def second(D, lab):
    s2 = D.clone()
    s2.scatter_(1, lab[:, None], float("inf"))
    return s2.min(1).values


D = torch.cdist(F, C)
lab = D.argmin(1)
u = D[ar, lab].clone()
lb = second(D, lab)
u2, lb2 = u.clone(), lb.clone()
out = []
for it in range(a.iters):
    sums = torch.zeros_like(C).index_add_(0, lab, F)
    cnt = torch.bincount(lab, minlength=k).clamp(min=1).to(F.dtype)
    Cn = sums / cnt[:, None]
    delta = (Cn - C).norm(dim=1)
    C = Cn
    D = torch.cdist(F, C)
    new = D.argmin(1)
    cc = torch.cdist(C, C)
    cc.fill_diagonal_(float("inf"))
    shalf = 0.5 * cc.min(1).values
    dmax = delta.max()
    exact_u = D[ar, lab]
    exact_l = second(D, new)
    # plain Hamerly (device plan)
    u = u + delta[lab]
    lb = lb - dmax
    cand = u > torch.maximum(lb, shalf[lab])
    u = torch.where(cand, D[ar, new], u)
    lb = torch.where(cand, exact_l, lb)
    # with ub tightening first
    u2 = u2 + delta[lab]
    lb2 = lb2 - dmax
    fail = u2 > torch.maximum(lb2, shalf[lab])
    u2 = torch.where(fail, exact_u, u2)
    cand2 = u2 > torch.maximum(lb2, shalf[lab])
    u2 = torch.where(cand2, D[ar, new], u2)
    lb2 = torch.where(cand2, exact_l, lb2)
    moved = int((new != lab).sum().item())
    out.append((it, round(cand.float().mean().item(), 4), round(fail.float().mean().item(), 4),
                round(cand2.float().mean().item(), 4), moved))
    lab = new
print(json.dumps({"cols": "iter, hamerly candidates, tightened rows, candidates after tightening, moved",
                  "per_iter": out[:4] + out[4::8] + out[-2:]}))
