"""Host-driven pruned Lloyd iterations (csc_kmeans_iterate per call) at cfg2 scale,
so a launch list shows every kernel of an iteration (the loop graph's body is
not listed by ncu's per-kernel mode)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1706_03591_b200 import _native  # noqa: E402
from paper_1706_03591_b200._device import ptr, row_stride, stream  # noqa: E402
from paper_1706_03591_b200.kmeans import _Workspace  # noqa: E402

n, d, k = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (20000, 80, 20)))
g = torch.Generator(device="cuda").manual_seed(0)
centers = torch.randn((k, d), dtype=torch.float64, device="cuda", generator=g) * 0.3
lab = torch.randint(0, k, (n,), device="cuda", generator=g)
blk = torch.zeros((n, row_stride(d)), dtype=torch.float64, device="cuda")
blk[:, :d] = centers[lab] + torch.randn((n, d), dtype=torch.float64, device="cuda", generator=g) * 0.2
ws = _Workspace(blk, d, k)
ws.cent[:, :d] = blk[torch.randperm(n, device="cuda", generator=g)[:k], :d]
_native.call("csc_kmeans_rownorms", ptr(ws.blk), n, d, ws.ld, ptr(ws.fnorm), stream())
history = []
cost = ws._lloyd_pruned(30, 0.0, history)
torch.cuda.synchronize()
print(f"n={n} d={d} k={k}: {len(history)} iterations, cost {cost:.6f}")
