"""Per-kernel times of host-driven pruned Lloyd iterations with and without the FP32 screen (torch.profiler)."""
import collections
import ctypes
import importlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1706_03591_b200 as P  # noqa: E402
from paper_1706_03591_b200 import _native  # noqa: E402
from paper_1706_03591_b200 import generators as G  # noqa: E402
from paper_1706_03591_b200._device import ptr, stream  # noqa: E402
from paper_1706_03591_b200.filters import FilteredBlock, _search_cutoff  # noqa: E402
from paper_1706_03591_b200.signals import device_signals  # noqa: E402

KM = importlib.import_module("paper_1706_03591_b200.kmeans")
n, k, d, m = 2_000_000, 64, 96, 80
q1, q2 = G.sbm_probabilities(n, k, 20.0, 0.05)
g = G.graph_from_codes(n, G.planted_partition_codes(n, k, q1, q2, 5))
lap = P.laplacian(g)
blk = device_signals(n, d, 0)
cut, filt, poly, iters, est = _search_cutoff(lap, k, FilteredBlock(blk, d), (0.0, 2.0),
                                             P.FilterConfig(order=m), None, 1.0)
F = filt.blk
ws = KM._Workspace(F, d, k)
seeds = KM.batched_kmeanspp(ws, np.random.SeedSequence(1).spawn(1))
plan = ws._plan()
ld32 = (d + 3) // 4 * 4
F32 = torch.zeros((n, ld32), dtype=torch.float32, device=F.device)
fn32 = torch.empty(n, dtype=torch.float32, device=F.device)
_native.call("csc_kmeans_screen_prepare", ptr(F), n, d, F.shape[1], ptr(F32), ld32, ptr(fn32), stream())
import sys as _sys  # noqa: E402
ITERS = int(_sys.argv[1]) if len(_sys.argv) > 1 else 40
MODES = _sys.argv[2].split(",") if len(_sys.argv) > 2 else ["fp64", "simt", "tc", "tc_full_update"]
for mode in MODES:
    _native.call("csc_kmeans_tuning", b"screen_tc", 1 if mode.startswith("tc") else 0)
    _native.call("csc_kmeans_tuning", b"update_incremental", 0 if mode == "tc_full_update" else 1)
    if mode == "fp64":
        _native.call("csc_kmeans_plan_set_screen", plan, None, 0, None)
    else:
        _native.call("csc_kmeans_plan_set_screen", plan, ptr(F32), ld32, ptr(fn32))
    ws.cent.copy_(seeds[0])
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        c2 = ws.lloyd(ITERS, 1e-6)
        torch.cuda.synchronize()
    tot = collections.defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            tot[e.name[:60]][0] += 1
            tot[e.name[:60]][1] += e.time_range.elapsed_us()
    total = sum(v[1] for v in tot.values())
    print(f"mode={mode}: cost2 {c2!r}  GPU total {total / 1e3:.2f} ms over {ITERS} iterations")
    for name, (c, us) in sorted(tot.items(), key=lambda x: -x[1][1])[:10]:
        print(f"   {us:9.1f} us x{c:4d}  {name}")
    seq = collections.defaultdict(list)
    for e in sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
                    key=lambda e: e.time_range.start):
        for key in ("update_sorted", "fx_delta", "fx_sum", "fx_scatter", "fx_changes", "screen_kernel",
                    "assign3", "assign_small", "finish_small"):
            if key in e.name:
                seq[key].append(round(e.time_range.elapsed_us()))
                break
    for key, v in seq.items():
        print(f"   per-iteration {key}: {v[:6]} ... {v[-6:]}")

# label changes per iteration (host diff of the labels after each iteration) and
# the fraction of (chunk, cluster) partial sums they dirty (chunk = the plan's)
if "changes" in MODES:
    _native.call("csc_kmeans_tuning", b"screen_tc", 1)
    _native.call("csc_kmeans_plan_set_screen", plan, ptr(F32), ld32, ptr(fn32))
    ws.cent.copy_(seeds[0])
    _native.call("csc_kmeans_rownorms", ptr(ws.cent), k, d, ws.ldc, ptr(ws.cnorm), stream())
    ws.labels.zero_()
    nb = max(1, min(148 * 8, -(-n // 64)))
    chunk = -(-n // nb)
    prev = None
    out = []
    for it in range(ITERS):
        _native.call("csc_kmeans_iterate", plan, ptr(ws.blk), ptr(ws.fnorm), ptr(ws.cent), ws.ldc, ptr(ws.cnorm),
                     ptr(ws.labels), ptr(ws.counts), int(it == 0), ptr(ws.scalars[1:]), stream())
        lab = ws.labels.cpu().numpy().astype(np.int64)
        cand = ctypes.c_int64()
        _native.call("csc_kmeans_plan_stats", plan, ctypes.byref(cand), None)
        amb = ctypes.c_int64()
        _native.call("csc_kmeans_plan_screen_stats", plan, ctypes.byref(amb))
        if prev is not None:
            ch = np.flatnonzero(lab != prev)
            blocks = ch // chunk
            pairs = np.unique(np.concatenate([blocks * k + lab[ch], blocks * k + prev[ch]]))
            out.append((it, ch.size, pairs.size / (nb * k), cand.value, amb.value))
        prev = lab
    for it, c, frac, cd, am in out[::max(1, len(out) // 12)]:
        print(f"   iter {it}: {c} rows changed, dirty (chunk, cluster) fraction {frac:.3f}, "
              f"Hamerly candidates {cd}, undecided by the screen {am}")
