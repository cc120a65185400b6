"""Interleaved A/B of k-means assignment kernel versions (CUDA events)."""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1706_03591_b200 import _native  # noqa: E402
from paper_1706_03591_b200._device import ptr, row_stride, stream  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2_000_000)
ap.add_argument("--d", type=int, default=96)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--rounds", type=int, default=7)
a = ap.parse_args()
lib = _native.lib()
ld = row_stride(a.d)
g = torch.Generator(device="cuda").manual_seed(0)
f = torch.zeros((a.n, ld), dtype=torch.float64, device="cuda")
f[:, :a.d] = torch.randn((a.n, a.d), dtype=torch.float64, device="cuda", generator=g)
c = torch.zeros((a.k, ld), dtype=torch.float64, device="cuda")
c[:, :a.d] = torch.randn((a.k, a.d), dtype=torch.float64, device="cuda", generator=g)
fn = (f * f).sum(1)
cn = (c * c).sum(1)
VARIANTS = [("v2", "assign_ver", 2), ("small", "assign_tile", 1), ("v3-88", "assign_tile", 88), ("v3-84", "assign_tile", 84), ("v3-87", "assign_tile", 87),
            ("v3-48", "assign_tile", 48),
            ("v3-44", "assign_tile", 44), ("v3-42", "assign_tile", 42)]
if a.k > 64 or a.d > 128:
    VARIANTS = [v for v in VARIANTS if v[0] != "small"]
labels = {v[0]: torch.empty(a.n, dtype=torch.int32, device="cuda") for v in VARIANTS}
own = torch.empty(a.n, dtype=torch.float64, device="cuda")
counts = torch.empty(a.k, dtype=torch.int32, device="cuda")
times = {v[0]: [] for v in VARIANTS}
for r in range(a.rounds):
    for name, key, val in VARIANTS:
        v = name
        _native.check(lib.csc_kmeans_tuning(b"assign_ver", 2 if name == "v2" else 3), "tuning")
        if key == "assign_tile":
            _native.check(lib.csc_kmeans_tuning(b"assign_tile", val), "tuning")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _native.call("csc_kmeans_assign", ptr(f), ptr(fn), a.n, a.d, ld, ptr(c), ld, ptr(cn), a.k,
                     ptr(labels[v]), ptr(own), ptr(counts), stream())
        e1.record()
        torch.cuda.synchronize()
        if r:
            times[v].append(e0.elapsed_time(e1))
flop = 2.0 * a.n * a.k * a.d
for v, _, _ in VARIANTS:
    m = statistics.median(times[v])
    print(f"assign {v}: n={a.n} d={a.d} k={a.k} median {m:.3f} ms ({flop / m / 1e9:.1f} TFLOP/s) "
          f"min {min(times[v]):.3f} max {max(times[v]):.3f}")
_native.check(lib.csc_kmeans_tuning(b"assign_tile", 0), "tuning")
print("labels equal:", all(bool(torch.equal(labels["v2"], labels[v[0]])) for v in VARIANTS))
