"""Interleaved in-process A/B of csc_kmeans_assign across library builds (CUDA events).

    python tools/ab_libs.py libA.so libB.so ... [--n 2000000 --d 96 --k 64 --rounds 9]
"""
import argparse
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1706_03591_b200 import _native  # noqa: E402
from paper_1706_03591_b200._device import ptr, row_stride, stream  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--n", type=int, default=2_000_000)
ap.add_argument("--d", type=int, default=96)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--rounds", type=int, default=9)
ap.add_argument("--no-counts", action="store_true")
a = ap.parse_args()
libs = []
for path in a.libs:
    lib = ctypes.CDLL(os.path.abspath(path), mode=ctypes.RTLD_LOCAL)
    args, res = _native.SIGNATURES["csc_kmeans_assign"]
    lib.csc_kmeans_assign.argtypes, lib.csc_kmeans_assign.restype = args, res
    libs.append(lib)
ld = row_stride(a.d)
g = torch.Generator(device="cuda").manual_seed(0)
f = torch.zeros((a.n, ld), dtype=torch.float64, device="cuda")
f[:, :a.d] = torch.randn((a.n, a.d), dtype=torch.float64, device="cuda", generator=g)
c = torch.zeros((a.k, ld), dtype=torch.float64, device="cuda")
c[:, :a.d] = torch.randn((a.k, a.d), dtype=torch.float64, device="cuda", generator=g)
fn = (f * f).sum(1)
cn = (c * c).sum(1)
labels = [torch.empty(a.n, dtype=torch.int32, device="cuda") for _ in libs]
own = torch.empty(a.n, dtype=torch.float64, device="cuda")
counts = torch.empty(a.k, dtype=torch.int32, device="cuda")
times = [[] for _ in libs]
for r in range(a.rounds):
    for i, lib in enumerate(libs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = lib.csc_kmeans_assign(ptr(f), ptr(fn), a.n, a.d, ld, ptr(c), ld, ptr(cn), a.k, ptr(labels[i]),
                                   ptr(own), None if a.no_counts else ptr(counts), stream())
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0, rc
        if r:
            times[i].append(e0.elapsed_time(e1))
flop = 2.0 * a.n * a.k * a.d
for path, t in zip(a.libs, times):
    m = statistics.median(t)
    print(f"{os.path.basename(path)}: n={a.n} d={a.d} k={a.k} median {m:.3f} ms ({flop / m / 1e9:.1f} TFLOP/s) "
          f"min {min(t):.3f} max {max(t):.3f}")
print("labels equal:", all(bool(torch.equal(labels[0], x)) for x in labels))
