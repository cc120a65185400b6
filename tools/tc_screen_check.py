"""Numerics and timing of the tcgen05 (kind::tf32, 3xTF32) screen's distances (tools only).

    python tools/tc_screen_check.py [--n 200000 --d 96 --k 64]

E_tc (csc_kmeans_tc_distances) against the exact fp64 GEMM-form distances:
max |E_tc - D| / (|f| + max|c|)^2 against the screen's bound (3d + 8) 2^-23,
first-argmin agreement, and CUDA-event time per call on n rows.
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_03591_b200 import _native  # noqa: E402
from paper_1706_03591_b200._device import ptr, stream  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=200_000)
ap.add_argument("--d", type=int, default=96)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
n, d, k = a.n, a.d, a.k
g = torch.Generator(device="cuda").manual_seed(1)
# clustered features like CSC's: centroids + small noise
cent = torch.randn((k, d), dtype=torch.float64, device="cuda", generator=g) / np.sqrt(d)
lab = torch.randint(0, k, (n,), device="cuda", generator=g)
f64 = cent[lab] + 0.3 * torch.randn((n, d), dtype=torch.float64, device="cuda", generator=g) / np.sqrt(d)
c64 = cent + 0.05 * torch.randn((k, d), dtype=torch.float64, device="cuda", generator=g) / np.sqrt(d)
ld32 = (d + 3) // 4 * 4
f32 = torch.zeros((n, ld32), dtype=torch.float32, device="cuda")
f32[:, :d] = f64.float()
fn32 = (f32.double() ** 2).sum(1).float()
cnorm = (c64 ** 2).sum(1)
npad = (k + 15) // 16 * 16
E = torch.empty((n, npad), dtype=torch.float32, device="cuda")
_native.call("csc_kmeans_tc_distances", ptr(f32), n, d, ld32, ptr(fn32), ptr(c64), k, d, ptr(cnorm), ptr(E), stream())
torch.cuda.synchronize()
D = (f64 ** 2).sum(1, keepdim=True) - 2 * f64 @ c64.T + cnorm[None, :]
Et = E[:, :k].double()
scale = (f64.norm(dim=1, keepdim=True) + cnorm.sqrt().max()) ** 2
err = ((Et - D).abs() / scale).max().item()
bound = (3 * d + 8) * 2.0 ** -23
agree = (Et.argmin(1) == D.argmin(1)).float().mean().item()
print(f"max |E_tc - D| / (|f|+cmax)^2 = {err:.3e}  bound {bound:.3e}  ratio {err / bound:.3f}  "
      f"argmin agreement {agree:.6f}", flush=True)
srt = D.sort(1).values
gap = (srt[:, 1] - srt[:, 0]) / scale[:, 0]
print(f"rows decided at the bound (gap > 2 delta): {(gap > 2 * bound).float().mean().item():.4f}; "
      f"at the FP32-screen bound {(gap > 2 * (d + 5) * 2.0 ** -24).float().mean().item():.4f}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    _native.call("csc_kmeans_tc_distances", ptr(f32), n, d, ld32, ptr(fn32), ptr(c64), k, d, ptr(cnorm), ptr(E),
                 stream())
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
print(f"tc distances: {ms:.3f} ms per call on {n} rows ({n * d * 4 / ms / 1e6:.1f} GB/s of F32 rows, "
      f"incl. writing E {n * npad * 4 / 1e6:.0f} MB)")
assert err <= bound, "bound violated"
