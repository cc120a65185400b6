"""Row-candidate fraction of Hamerly vs Yinyang-style group bounds on real
cfg5 features (tools only). Exact Lloyd in torch fp64; bounds kept the way a
device plan would (candidates get exact bounds from a full evaluation, the
other rows propagate them): Hamerly's one lower bound relaxed by the largest
centroid movement, and t group lower bounds each relaxed by its group's own
largest movement (centroid groups: k-means of the seeds, as Yinyang does).

    python tools/yinyang_sim.py [--groups 8 --iters 100]
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
ap.add_argument("--groups", type=int, default=8)
ap.add_argument("--iters", type=int, default=100)
a = ap.parse_args()
n, k, d, m = 2_000_000, 64, 96, 80
g, _ = G.planted_partition_device(n, k, 20.0, 0.05, seed=5)
lap = P.laplacian(g)
blk = device_signals(n, d, 0)
cut, filt, poly, iters, est = _search_cutoff(lap, k, FilteredBlock(blk, d), (0.0, 2.0), P.FilterConfig(order=m),
                                             None, 1.0)
ws = _Workspace(filt.blk, d, k)
seeds = batched_kmeanspp(ws, np.random.SeedSequence(1).spawn(1))
F = filt.blk[:, :d].contiguous()
C = seeds[0][:, :d].clone()
ar = torch.arange(n, device=F.device)
t = a.groups
# centroid groups: a few Lloyd steps on the seeds themselves
gc = C[torch.randperm(k, device=F.device)[:t]].clone()
for _ in range(10):
    grp = torch.cdist(C, gc).argmin(1)
    for q in range(t):
        if (grp == q).any():
            gc[q] = C[grp == q].mean(0)
grp = torch.cdist(C, gc).argmin(1)
ginf = torch.full((k,), float("inf"), dtype=F.dtype, device=F.device)


def group_mins(D, lab):
    D2 = D.clone()
    D2[ar, lab] = float("inf")
    return torch.stack([D2[:, grp == q].min(1).values if (grp == q).any() else ginf[:n] for q in range(t)], 1)


D = torch.cdist(F, C)
lab = D.argmin(1)
u = D[ar, lab].clone()
lbh = group_mins(D, lab).min(1).values
lbg = group_mins(D, lab)
uy = u.clone()
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
    gm = group_mins(D, new)
    # Hamerly
    u = u + delta[lab]
    lbh = lbh - delta.max()
    cand_h = u > torch.maximum(lbh, shalf[lab])
    u = torch.where(cand_h, D[ar, new], u)
    lbh = torch.where(cand_h, gm.min(1).values, lbh)
    # Yinyang-style group bounds (row filter only)
    gd = torch.stack([delta[grp == q].max() if (grp == q).any() else delta.new_zeros(()) for q in range(t)])
    uy = uy + delta[lab]
    lbg = lbg - gd[None, :]
    cand_y = uy > torch.maximum(lbg.min(1).values, shalf[lab])
    uy = torch.where(cand_y, D[ar, new], uy)
    lbg = torch.where(cand_y[:, None], gm, lbg)
    out.append((it, round(cand_h.float().mean().item(), 4), round(cand_y.float().mean().item(), 4),
                int((new != lab).sum().item())))
    lab = new
print(json.dumps({"groups": t, "cols": "iter, hamerly candidates, yinyang candidates, moved",
                  "mean_h": round(float(np.mean([o[1] for o in out])), 4),
                  "mean_y": round(float(np.mean([o[2] for o in out])), 4),
                  "per_iter": out[:4] + out[4::12] + out[-2:]}))
