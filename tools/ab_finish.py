"""A/B of the Lloyd iteration tail variants (csc_kmeans_tuning finish_mode) at
cfg2 scale: per-iteration time of one host-driven pruned Lloyd run (CUDA events)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1706_03591_b200 import _native  # noqa: E402
from paper_1706_03591_b200._device import ptr, row_stride, stream  # noqa: E402
from paper_1706_03591_b200.kmeans import _Workspace  # noqa: E402

n, d, k = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (20000, 80, 20)))
lib = _native.lib()
g = torch.Generator(device="cuda").manual_seed(0)
centers = torch.randn((k, d), dtype=torch.float64, device="cuda", generator=g) * 0.3
lab = torch.randint(0, k, (n,), device="cuda", generator=g)
blk = torch.zeros((n, row_stride(d)), dtype=torch.float64, device="cuda")
blk[:, :d] = centers[lab] + torch.randn((n, d), dtype=torch.float64, device="cuda", generator=g) * 0.2
seed = blk[torch.randperm(n, device="cuda", generator=g)[:k], :d].clone()
ws = _Workspace(blk, d, k)
_native.call("csc_kmeans_rownorms", ptr(ws.blk), n, d, ws.ld, ptr(ws.fnorm), stream())
plan = ws._plan()
times = {m: [] for m in (0, 1, 2)}
results = {}
for rep in range(6):
    for m in (0, 1, 2):
        _native.check(lib.csc_kmeans_tuning(b"finish_mode", m), "tuning")
        ws.cent[:, :d] = seed
        _native.call("csc_kmeans_rownorms", ptr(ws.cent), k, d, ws.ldc, ptr(ws.cnorm), stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for it in range(20):
            _native.call("csc_kmeans_iterate", plan, ptr(ws.blk), ptr(ws.fnorm), ptr(ws.cent), ws.ldc,
                         ptr(ws.cnorm), ptr(ws.labels), ptr(ws.counts), int(it == 0), ptr(ws.scalars[1:]),
                         stream())
        e1.record()
        torch.cuda.synchronize()
        if rep:
            times[m].append(e0.elapsed_time(e1) / 20 * 1e3)
        results[m] = (ws.labels.clone(), ws.cent.clone())
_native.check(lib.csc_kmeans_tuning(b"finish_mode", 0), "tuning")
for m in (0, 1, 2):
    print(f"finish_mode {m}: {statistics.median(times[m]):.1f} us/iteration (host-launched, 20 iterations)")
print("labels equal:", all(torch.equal(results[0][0], results[m][0]) for m in (1, 2)),
      "centroids equal:", all(torch.equal(results[0][1], results[m][1]) for m in (1, 2)))
