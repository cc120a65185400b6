"""k-means kernels at tile / chunk / kernel-variant boundaries (GPU).

compute-sanitizer is not available on the GPU pool, so out-of-bounds and
ragged-edge mistakes are hunted here instead: every assignment kernel variant
(small-k, v2, and each v3 register tile) over shapes straddling its tile
sizes, pruned vs full Lloyd iterations over chunk boundaries of the
label-sorted update, and the update against numpy means with empty clusters.
Reference semantics: kmeans.py:54-61 (GEMM-form distances, first argmin),
kmeans.py:80-85 (means by label), kmeans.py:96-111 (Lloyd iteration).
"""
import numpy as np
import pytest

from oracle import csc_oracle as O

pytestmark = pytest.mark.gpu

# (n, d, k): around the 32 / 64 / 112 / 128 centroid tiles, the 128-row tile,
# d around the 16-wide k-step and the small kernel's d <= 128 limit
ASSIGN_SHAPES = [(1, 1, 1), (7, 3, 2), (129, 5, 31), (1000, 17, 32), (1000, 24, 33), (2049, 8, 64),
                 (3001, 40, 65), (5000, 12, 100), (4097, 30, 112), (4097, 30, 113), (3000, 129, 70),
                 (600, 300, 250), (257, 16, 128), (255, 1, 129),
                 # wide d: the resident centroid tile no longer fits (streamed-centroid variant)
                 (700, 401, 100), (300, 1001, 7), (513, 2000, 65),
                 # k above the shared-memory label histogram
                 (3000, 4, 9000)]
# (tuning key, value) pairs; each must give the auto choice's labels bit for bit
VARIANTS = [("assign_tile", 1), ("assign_tile", 44), ("assign_tile", 88), ("assign_tile", 84),
            ("assign_tile", 87), ("assign_tile", 48), ("assign_tile", 42), ("assign_ver", 2)]


@pytest.fixture(scope="module")
def K(cuda_ok):
    import torch
    from paper_1706_03591_b200 import _native
    from paper_1706_03591_b200._device import ptr, row_stride, stream, upload_block
    return torch, _native, ptr, row_stride, stream, upload_block


def _reset(_native):
    _native.call("csc_kmeans_tuning", b"assign_tile", 0)
    _native.call("csc_kmeans_tuning", b"assign_ver", 3)
    _native.call("csc_kmeans_tuning", b"assign_tn", 8)


def _blobs(n, d, k, seed, spread=4.0):
    rng = np.random.default_rng(seed)
    centers = rng.normal(0.0, spread, (max(k, 1), d))
    return centers[rng.integers(max(k, 1), size=n)] + rng.normal(size=(n, d)), rng


def _assign(K, f, c):
    torch, _native, ptr, row_stride, stream, upload_block = K
    n, d = f.shape
    k = c.shape[0]
    fb = upload_block(f)
    cb = upload_block(c)
    fn = torch.empty(n, dtype=torch.float64, device="cuda")
    cn = torch.empty(k, dtype=torch.float64, device="cuda")
    _native.call("csc_kmeans_rownorms", ptr(fb), n, d, fb.shape[1], ptr(fn), stream())
    _native.call("csc_kmeans_rownorms", ptr(cb), k, d, cb.shape[1], ptr(cn), stream())
    labels = torch.full((n,), -7, dtype=torch.int32, device="cuda")
    own = torch.full((n,), np.nan, dtype=torch.float64, device="cuda")
    counts = torch.full((k,), -7, dtype=torch.int32, device="cuda")
    _native.call("csc_kmeans_assign", ptr(fb), ptr(fn), n, d, fb.shape[1], ptr(cb), cb.shape[1], ptr(cn), k,
                 ptr(labels), ptr(own), ptr(counts), stream())
    return labels.cpu().numpy(), own.cpu().numpy(), counts.cpu().numpy()


@pytest.mark.parametrize("n,d,k", ASSIGN_SHAPES)
def test_assign_variants_agree_and_are_exact(K, n, d, k):
    _native = K[1]
    f, rng = _blobs(n, d, k, 1000 + n + k)
    c = f[rng.choice(n, k, replace=k > n)] + 0.25 * rng.normal(size=(k, d))
    _reset(_native)
    try:
        lab, own, cnt = _assign(K, f, c)
        d2 = O.sq_dists(f, c)
        srt = np.sort(d2, axis=1)
        clear = (srt[:, 1] - srt[:, 0]) > 1e-9 * (1.0 + srt[:, 0]) if k > 1 else np.ones(n, bool)
        assert lab.min() >= 0 and lab.max() < k
        assert np.array_equal(lab[clear], d2.argmin(1)[clear])
        scale = (f * f).sum(1) + (c * c).sum(1)[lab]
        assert np.all(np.abs(own - d2[np.arange(n), lab]) <= 1e-12 * (1.0 + scale))
        assert np.array_equal(cnt, np.bincount(lab, minlength=k))
        for key, val in VARIANTS:
            if key == "assign_tile" and val == 1 and not (k <= 64 and d <= 128):
                continue
            _reset(_native)
            _native.call("csc_kmeans_tuning", key.encode(), val)
            lab2, own2, cnt2 = _assign(K, f, c)
            # tuning knobs are performance-only: identical distances, labels, counts
            assert np.array_equal(lab2, lab), (key, val)
            assert np.array_equal(own2, own), (key, val)
            assert np.array_equal(cnt2, cnt), (key, val)
    finally:
        _reset(_native)


# (n, d, k, duplicate seeds): n around the plan's 64-row chunk floor and the
# 1184-chunk cap, k around the tiles, duplicated seeds force empty clusters
LLOYD_SHAPES = [(1, 1, 1, False), (5, 2, 5, False), (300, 3, 33, True), (8191, 4, 64, False),
                (8193, 7, 65, True), (20000, 24, 100, False), (75777, 16, 113, False),
                (30000, 9, 130, True), (12345, 40, 17, False), (1184 * 64 + 1, 5, 8, False)]


def _lloyd_trace(K, ws, seeds, iters, full_always):
    torch, _native, ptr, row_stride, stream, upload_block = K
    s = stream()
    ws.cent.zero_()
    ws.cent[:, :ws.d] = torch.from_numpy(seeds).cuda()
    _native.call("csc_kmeans_rownorms", ptr(ws.cent), ws.k, ws.d, ws.ldc, ptr(ws.cnorm), s)
    ws.labels.zero_()
    plan = ws._plan()
    out = []
    for it in range(iters):
        _native.call("csc_kmeans_iterate", plan, ptr(ws.blk), ptr(ws.fnorm), ptr(ws.cent), ws.ldc, ptr(ws.cnorm),
                     ptr(ws.labels), ptr(ws.counts), int(full_always or it == 0), ptr(ws.scalars[1:]), s)
        out.append((ws.labels.cpu().numpy().copy(), ws.cent[:, :ws.d].cpu().numpy().copy(),
                    ws.counts.cpu().numpy().copy(), float(ws.scalars[1].item())))
    return out


@pytest.mark.parametrize("n,d,k,dup", LLOYD_SHAPES)
def test_pruned_iterations_equal_full_and_oracle(K, n, d, k, dup):
    from paper_1706_03591_b200.kmeans import _Workspace
    f, rng = _blobs(n, d, max(k // 2, 1), 7 * n + k, spread=2.0)
    seeds = f[rng.choice(n, k, replace=False)].copy()
    if dup and k >= 3:
        seeds[2] = seeds[1]
    blk = K[5](f)
    iters = 6
    pruned = _lloyd_trace(K, _Workspace(blk, d, k), seeds, iters, False)
    full = _lloyd_trace(K, _Workspace(blk, d, k), seeds, iters, True)
    for it, ((la, ca, na, sa), (lb, cb, nb, sb)) in enumerate(zip(pruned, full)):
        assert np.array_equal(la, lb), it
        assert np.array_equal(ca, cb), it
        assert np.array_equal(na, nb), it
        assert sa == sb, it
        assert np.array_equal(na, np.bincount(la, minlength=k)) and na.min() >= 1
        sums = np.zeros((k, d))
        np.add.at(sums, la, f)
        assert np.allclose(ca, sums / na[:, None], rtol=1e-12, atol=1e-12 * np.abs(f).max())
    ol, oc2, _, oit = O.lloyd(f, k, seeds, iters, 0.0)  # tol 0: stops only on no improvement
    lab_o, _, _, c2_o = pruned[oit - 1]
    assert np.array_equal(lab_o, ol) if n < 2 else O.adjusted_rand(lab_o, ol) >= 0.999
    assert abs(c2_o - oc2) <= 1e-9 * max(oc2, 1e-300) + 1e-12


@pytest.mark.parametrize("n,d,k", [(1, 1, 1), (100, 3, 7), (5000, 33, 64), (20001, 8, 150), (4096, 300, 20)])
def test_update_means_with_empty_clusters(K, n, d, k):
    torch, _native, ptr, row_stride, stream, upload_block = K
    rng = np.random.default_rng(n + d + k)
    f = rng.normal(size=(n, d))
    lab = rng.integers(0, max(k // 2, 1), size=n).astype(np.int32)  # upper half of clusters empty
    fb = upload_block(f)
    ldc = row_stride(d)
    c = torch.full((k, ldc), np.nan, dtype=torch.float64, device="cuda")
    cn = torch.empty(k, dtype=torch.float64, device="cuda")
    cnt = torch.full((k,), -1, dtype=torch.int32, device="cuda")
    labels = torch.from_numpy(lab).cuda()
    _native.call("csc_kmeans_update", ptr(fb), ptr(labels), n, d, fb.shape[1], k, ptr(c), ldc, ptr(cn), ptr(cnt),
                 stream())
    counts = np.bincount(lab, minlength=k)
    sums = np.zeros((k, d))
    np.add.at(sums, lab, f)
    want = sums / np.maximum(counts, 1)[:, None]
    got = c[:, :d].cpu().numpy()
    assert np.array_equal(cnt.cpu().numpy(), counts)
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12 * np.abs(f).max())
    assert np.all(got[counts == 0] == 0.0)
    assert np.allclose(cn.cpu().numpy(), (got * got).sum(1), rtol=1e-12, atol=1e-300)


@pytest.mark.parametrize("d", [400, 1000])
def test_kmeans_wide_features_match_oracle(K, d):
    """Drop-in API at widths past every resident shared-memory tile (assign,
    batched k-means++, iteration tail): same clustering as the oracle."""
    import paper_1706_03591_b200 as P
    f, _ = _blobs(1500, d, 6, d, spread=0.3)
    a = P.kmeans(f, 6, P.KmeansConfig(restarts=3, max_iters=30), seed=5)
    lab, sizes, cost = O.kmeans(f, 6, restarts=3, max_iters=30, seed=5)
    assert O.adjusted_rand(a.labels, lab) >= 0.999
    assert np.array_equal(np.sort(a.cluster_sizes), np.sort(sizes))
    assert abs(a.feature_cost - cost) <= 1e-9 * cost
