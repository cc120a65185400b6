"""One k-means assignment at cfg5 scale for ncu (n=2M, d=96, k=64)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_03591_b200._device import row_stride  # noqa: E402
from paper_1706_03591_b200.kmeans import _Workspace  # noqa: E402

n, d, k = int(os.environ.get("N", 2_000_000)), int(os.environ.get("D", 96)), int(os.environ.get("K", 64))
g = torch.Generator(device="cuda").manual_seed(0)
blk = torch.zeros((n, row_stride(d)), dtype=torch.float64, device="cuda")
blk[:, :d] = torch.randn((n, d), dtype=torch.float64, device="cuda", generator=g)
ws = _Workspace(blk, d, k)
ws.kmeanspp(np.random.default_rng(0))
ws.lloyd(2, 0.0)
torch.cuda.synchronize()
print("ok")
