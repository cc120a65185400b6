"""Phase split of one end-to-end apply_filter call at cfg3 (numpy pinned in, numpy out)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import generators as G  # noqa: E402
from paper_1706_03591_b200._device import download_block, upload_block  # noqa: E402
from paper_1706_03591_b200.filters import filter_block  # noqa: E402

n, k, d, m = 1_000_000, 100, 128, 100
q1, q2 = G.sbm_probabilities(n, k, 32.0, 0.02)
lap = P.laplacian(G.graph_from_codes(n, G.planted_partition_codes(n, k, q1, q2, 3)))
poly = P.cheb_coeffs(0.6, lap.lambda_max_bound, m)
x_np = torch.randn((n, d), dtype=torch.float64).pin_memory().numpy()
P.apply_filter(lap, poly, x_np)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    res = P.apply_filter(lap, poly, x_np)
    torch.cuda.synchronize()
    total = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    blk = upload_block(x_np)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    out, _ = filter_block(lap, poly, blk, d)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    h = download_block(out, d)
    t3 = time.perf_counter()
    print(f"apply_filter {total:.1f} ms | upload {(t1 - t0) * 1e3:.1f} filter {(t2 - t1) * 1e3:.1f} "
          f"download {(t3 - t2) * 1e3:.1f} ms")
    del res, h, out, blk

# host pipelines: column chunks (round 1) vs row slices (download overlapped
# with the last order), pinned and pageable input
from paper_1706_03591_b200 import filters as PF  # noqa: E402
ref = P.apply_filter(lap, poly, torch.from_numpy(x_np).cuda()).cpu().numpy()
x_pg = np.array(x_np)
variants = [("columns", 2, 0), ("slices", 1, 8), ("slices", 4, 8), ("slices", 8, 8), ("slices", 16, 16)]
for rnd in range(2):
    for mode, sl, up in variants:
        PF.PIPE_MODE, PF.PIPE_CHUNKS, PF.PIPE_SLICES, PF.PIPE_UP_SLICES = mode, 2, sl, max(1, up)
        for name, xin in (("pinned", x_np), ("pageable", x_pg)):
            res = P.apply_filter(lap, poly, xin)
            ts = []
            for rep in range(4):
                t0 = time.perf_counter()
                res = P.apply_filter(lap, poly, xin)
                torch.cuda.synchronize()
                ts.append((time.perf_counter() - t0) * 1e3)
            same = bool(np.array_equal(res, ref))
            print(f"{mode:8s} slices {sl:2d} up {up:2d} {name:8s}: {min(ts):.1f} / {np.median(ts):.1f} ms "
                  f"(min / median), bitwise equal to the device path: {same}", flush=True)
