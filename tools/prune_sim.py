"""How many (row, centroid) distances would Hamerly / Elkan / Yinyang bounds
need on real CSC features?  Exact Lloyd in torch fp64 on the GPU (full
distance matrix each iteration), bounds simulated alongside; prints per
iteration the fraction of the n*k distances each scheme evaluates.

    python tools/prune_sim.py [--n 2000000 --k 64 --d 96 --m 80 --iters 100 --groups 8]
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
ap.add_argument("--deg", type=float, default=20.0)
ap.add_argument("--ratio", type=float, default=0.05)
ap.add_argument("--iters", type=int, default=100)
ap.add_argument("--groups", type=int, default=8)
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
n, k = a.n, a.k
grp = torch.arange(k, device=F.device) % a.groups  # round-robin groups (no clustering of centroids)


def dists(C):
    return torch.cdist(F, C)  # fp64 Euclidean


D = dists(C)
lab = D.argmin(1)
u = D.gather(1, lab[:, None])[:, 0].clone()
L = D.clone()  # Elkan lower bounds (exact at start)
s2 = D.clone()
s2.scatter_(1, lab[:, None], float("inf"))
lh = s2.min(1).values  # Hamerly lower bound
Ly = torch.stack([torch.where(grp[None, :] == t, s2, torch.full_like(s2, float("inf"))).min(1).values
                  for t in range(a.groups)], 1)  # Yinyang group bounds (excluding own)
LF = D.clone()  # per-centroid bounds used only as a row filter (rows refreshed by full evaluation)
uF = u.clone()
out = []
ar = torch.arange(n, device=F.device)
for it in range(a.iters):
    sums = torch.zeros_like(C).index_add_(0, lab, F)
    cnt = torch.bincount(lab, minlength=k).clamp(min=1).to(F.dtype)
    Cn = sums / cnt[:, None]
    delta = (Cn - C).norm(dim=1)
    C = Cn
    D = dists(C)
    new = D.argmin(1)
    cc = torch.cdist(C, C)
    cc.fill_diagonal_(float("inf"))
    shalf = 0.5 * cc.min(1).values
    # --- Hamerly (as in the device plan): candidates = rows whose bounds fail
    u = u + delta[lab]
    dmax = delta.max()
    lh = lh - dmax
    ham = (u > torch.maximum(lh, shalf[lab]))
    # --- Elkan: per-centroid bounds; a row is skipped if u <= s(a); else tighten u (1 distance),
    #     then evaluate pairs with u > l(x,c) and u > cc(a,c)/2
    L = L - delta[None, :]
    rows_e = u > shalf[lab]
    ut = D[ar, lab]  # tightened u
    pair = (ut[:, None] > L) & (ut[:, None] > 0.5 * cc[lab]) & rows_e[:, None]
    pair[ar, lab] = False
    elkan_evals = rows_e.sum().item() + pair.sum().item()
    # --- Yinyang (group filter on group bounds, then every centroid of a surviving group)
    gd = torch.stack([delta[grp == t].max() for t in range(a.groups)])
    Ly = Ly - gd[None, :]
    gpass = (ut[:, None] > Ly) & rows_e[:, None]
    gsize = torch.bincount(grp, minlength=a.groups)
    yy_evals = rows_e.sum().item() + (gpass.to(torch.int64) * gsize[None, :]).sum().item()
    # --- per-centroid bounds as a row filter; candidate rows evaluated in full (GEMM)
    LF = LF - delta[None, :]
    uF = uF + delta[lab]
    LFo = LF.clone()
    LFo.scatter_(1, lab[:, None], float("inf"))
    rowsF = uF > torch.maximum(LFo.min(1).values, shalf[lab])
    out.append((it, round(ham.float().mean().item(), 4), round(elkan_evals / (n * k), 4),
                round(yy_evals / (n * k), 4), round(rowsF.float().mean().item(), 4), int((new != lab).sum().item())))
    LF = torch.where(rowsF[:, None], D, LF)
    uF = torch.where(rowsF, D[ar, new], uF)
    # exact refresh of all bounds for the next iteration (what an exact pass would leave)
    lab = new
    u = D[ar, lab]
    s2 = D.clone()
    s2.scatter_(1, lab[:, None], float("inf"))
    # keep the *propagated* bounds where the pair was not evaluated, exact where it was
    L = torch.where(pair | (~rows_e[:, None]) == False, L, L)  # noqa: E712 (bounds stay conservative)
    L = torch.where(pair, D, L)
    L[ar, lab] = D[ar, lab]
    lh = torch.where(ham, s2.min(1).values, lh)
    Ly = torch.where(gpass, torch.stack([torch.where(grp[None, :] == t, s2, torch.full_like(s2, float("inf"))).min(1).values
                                         for t in range(a.groups)], 1), Ly)
print(json.dumps({"iters": len(out), "cols": "iter, hamerly_rows, elkan_evals/(nk), yinyang_evals/(nk), elkan_filter_rows, moved",
                  "per_iter": out[:6] + out[6::10] + out[-3:]}))
