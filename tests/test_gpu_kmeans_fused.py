"""Fused Lloyd (csc_kmeans_fused_run): every restart in one cooperative launch.

Parity bar (north_star): k-means started from the reference's initial
centroids gives ARI >= 0.999 and cost within 1e-9 relative. Each restart of
the fused launch is compared with the oracle's Lloyd (kmeans.py:88-117
restated) started from the same seeds; iteration counts must agree too.
"""
import numpy as np
import pytest

from conftest import golden
from oracle import csc_oracle as O

pytestmark = pytest.mark.gpu

COST_TOL = 1e-9


@pytest.fixture(scope="module")
def P(cuda_ok):
    import paper_1706_03591_b200 as P
    return P


def fused_run(f, k, seeds, max_iters=100, tol=1e-6):
    """Raw C-ABI call: seeds (R, k, d) host -> per-restart (labels, cost2, iters)."""
    import torch
    from paper_1706_03591_b200 import _native
    from paper_1706_03591_b200._device import ptr, row_stride, stream, upload_block
    blk = upload_block(np.ascontiguousarray(f, dtype=np.float64))
    n, ld = blk.shape
    d = f.shape[1]
    R = len(seeds)
    ldc = row_stride(d)
    dev = blk.device
    fn = torch.empty(n, dtype=torch.float64, device=dev)
    _native.call("csc_kmeans_rownorms", ptr(blk), n, d, ld, ptr(fn), stream())
    S = torch.zeros((R, k, ldc), dtype=torch.float64, device=dev)
    S[:, :, :d] = torch.from_numpy(np.stack(seeds).astype(np.float64)).to(dev)
    labels = torch.full((R, n), -7, dtype=torch.int32, device=dev)
    cost = torch.empty(R, dtype=torch.float64, device=dev)
    iters = torch.empty(R, dtype=torch.int32, device=dev)
    assert _native.lib().csc_kmeans_fused_supported(n, d, k, R, max_iters) == 1
    _native.call("csc_kmeans_fused_run", ptr(blk), ptr(fn), n, d, ld, k, R, ptr(S), ldc, int(max_iters),
                 float(tol), ptr(labels), ptr(cost), ptr(iters), stream())
    return labels.cpu().numpy().astype(np.int64), cost.cpu().numpy(), iters.cpu().numpy()


def check_against_oracle(f, k, seeds, max_iters=100, tol=1e-6, exact_labels=False):
    labels, cost, iters = fused_run(f, k, seeds, max_iters, tol)
    for r, c0 in enumerate(seeds):
        ref_labels, ref_cost2, _, ref_it = O.lloyd(f, k, c0, max_iters, tol)
        assert iters[r] == ref_it, (r, iters[r], ref_it)
        assert abs(cost[r] - ref_cost2) <= COST_TOL * ref_cost2, (r, cost[r], ref_cost2)
        if exact_labels:
            assert np.array_equal(labels[r], ref_labels), r
        else:
            assert O.adjusted_rand(labels[r], ref_labels) >= 0.999, r
    return labels, cost, iters


def blobs(n, d, k, spread, seed):
    rng = np.random.default_rng(seed)
    centers = rng.normal(size=(k, d))
    lab = rng.integers(0, k, n)
    return centers[lab] + spread * rng.normal(size=(n, d))


def pp_seeds(f, k, R, seed):
    return [O.kmeanspp(f, k, np.random.default_rng(c))[0] for c in np.random.SeedSequence(seed).spawn(R)]


def test_fused_cfg1_from_reference_init(P):
    """configs[0]: the reference's k-means++ seeds (golden), 20 iterations cap."""
    g = golden("cfg1")
    f = g["features"]
    labels, cost, iters = fused_run(f, 10, [g["km_init"]], max_iters=20)
    assert O.adjusted_rand(labels[0], g["km_labels"]) >= 0.999
    assert abs(cost[0] - float(g["km_cost2"])) <= COST_TOL * float(g["km_cost2"])
    assert iters[0] == len(g["km_hist"])


@pytest.mark.parametrize("n,d,k,R", [(20000, 80, 20, 6), (5000, 40, 10, 10), (3000, 128, 32, 3),
                                     (997, 7, 5, 16), (40, 3, 4, 2)])
def test_fused_restarts_match_oracle_lloyd(P, n, d, k, R):
    f = blobs(n, d, k, 0.8, seed=n + d)
    check_against_oracle(f, k, pp_seeds(f, k, R, seed=d))


def test_fused_iteration_cap_and_k1(P):
    f = blobs(2000, 16, 6, 1.5, seed=3)
    check_against_oracle(f, 6, pp_seeds(f, 6, 3, seed=1), max_iters=3, tol=0.0)
    labels, cost, iters = check_against_oracle(f, 1, pp_seeds(f, 1, 2, seed=2), exact_labels=True)
    assert (labels == 0).all() and iters[0] == 2  # k=1: the second cost repeats the first


def test_fused_empty_cluster_repair(P):
    """Seeds far from every row leave clusters empty on the first assignment:
    the reference reseeds each (ascending j) at the row farthest from its
    centroid (kmeans.py:99-108)."""
    rng = np.random.default_rng(5)
    f = rng.normal(size=(3000, 12))
    seeds = []
    for far in ([3], [1, 4], [0, 2, 5]):
        c = f[rng.choice(3000, 6, replace=False)].copy()
        for j in far:
            c[j] = 1e3 + 10.0 * j
        seeds.append(c)
    check_against_oracle(f, 6, seeds, exact_labels=True)


def test_fused_duplicate_rows_through_kmeans(P):
    """Zero D^2 mass in k-means++ (replayed) and empty clusters through the public kmeans()."""
    for s in range(6):
        b = P.kmeans(np.array([[0.0], [0.0], [5.0]]), 3, P.KmeansConfig(restarts=1), seed=s)
        assert b.cluster_sizes.min() >= 1
    f = np.repeat(np.arange(5.0)[:, None] * np.ones((1, 3)), 40, axis=0)
    a = P.kmeans(f, 7, P.KmeansConfig(restarts=4, max_iters=20), seed=9)
    ref_labels, _, ref_cost = O.kmeans(f, 7, restarts=4, max_iters=20, tol=1e-6, seed=9)
    assert a.cluster_sizes.min() >= 1
    assert abs(a.feature_cost - ref_cost) <= 1e-9 * max(ref_cost, 1e-300) + 1e-12


def test_fused_public_kmeans_matches_oracle(P):
    """kmeans() takes the fused path at configs[1]'s shape; best-of-restarts as the reference."""
    from paper_1706_03591_b200.kmeans import fused_supported
    f = blobs(20000, 80, 20, 1.0, seed=11)
    assert fused_supported(20000, 80, 20, 10, 100)
    a = P.kmeans(f, 20, seed=4)
    ref_labels, _, ref_cost = O.kmeans(f, 20, restarts=10, max_iters=100, tol=1e-6, seed=4)
    assert O.adjusted_rand(a.labels, ref_labels) >= 0.999
    assert abs(a.feature_cost - ref_cost) <= COST_TOL * ref_cost


def test_fused_equals_lanes(P):
    """Fused launch and per-restart lanes agree on the golden case (labels exactly, cost to 1e-9)."""
    from paper_1706_03591_b200._device import upload_block
    from paper_1706_03591_b200.kmeans import run_restarts
    g = golden("kmeans")
    blk = upload_block(g["b_f"])
    kids = np.random.SeedSequence(77).spawn(3)
    cfg = P.KmeansConfig(restarts=3, max_iters=50)
    lf, cf = run_restarts(blk, 24, 12, cfg, kids, fused=True)
    ll, cl = run_restarts(blk, 24, 12, cfg, kids, fused=False)
    assert np.array_equal(lf, ll)
    assert abs(cf - cl) <= COST_TOL * cl
    assert np.array_equal(lf, g["b_labels"])


def test_fused_shape_gate(P):
    from paper_1706_03591_b200.kmeans import fused_supported
    assert not fused_supported(20000, 80, 33, 10, 100)   # k > 32
    assert not fused_supported(20000, 129, 20, 10, 100)  # d > 128
    assert not fused_supported(2_000_000, 96, 20, 10, 100)  # rows exceed shared memory
    assert not fused_supported(20000, 80, 20, 10, 0)


def test_fused_kpp_seeds_match_reference_picks(P):
    """In-kernel k-means++ (csc_kmeans_fused_kpp_run): the seeds are the
    reference's picks for the same streams (kmeans.py:64-77), and every
    restart's Lloyd run then matches the oracle from those seeds."""
    import torch
    from paper_1706_03591_b200 import _native
    from paper_1706_03591_b200._device import ptr, row_stride, stream, upload_block
    from paper_1706_03591_b200.kmeans import kmeanspp_draws
    # restarts per distance item (kmeans_fused.cu kmeanspp_phase): 4 (997 rows),
    # 6 (20000 x R=10), 8 (20000 x R=13), back to 4 where 6 would pad past 32 (8000 x R=32)
    for n, d, k, R, seed in [(1000, 40, 10, 1, 0), (20000, 80, 20, 10, 5), (997, 7, 5, 16, 2),
                             (20000, 24, 6, 13, 3), (8000, 16, 8, 32, 4)]:
        f = blobs(n, d, k, 0.9, seed=seed)
        blk = upload_block(f)
        ld = blk.shape[1]
        ldc = row_stride(d)
        kids = np.random.SeedSequence(seed).spawn(R)
        first, unif = kmeanspp_draws(kids, n, k)
        dev = blk.device
        labels = torch.empty((R, n), dtype=torch.int32, device=dev)
        cost = torch.empty(R, dtype=torch.float64, device=dev)
        iters = torch.empty(R, dtype=torch.int32, device=dev)
        seeds = torch.zeros((R, k, ldc), dtype=torch.float64, device=dev)
        flags = torch.empty(R, dtype=torch.int32, device=dev)
        first = np.ascontiguousarray(first)
        unif = np.ascontiguousarray(unif)
        _native.call("csc_kmeans_fused_kpp_run", ptr(blk), n, d, ld, k, R, first.ctypes.data, unif.ctypes.data,
                     ldc, 100, 1e-6, ptr(labels), ptr(cost), ptr(iters), ptr(seeds), ptr(flags), stream())
        assert (flags.cpu().numpy() < 0).all()
        S = seeds[:, :, :d].cpu().numpy()
        lab, cst, its = labels.cpu().numpy(), cost.cpu().numpy(), iters.cpu().numpy()
        for r, child in enumerate(kids):
            ref_cent, ref_picks = O.kmeanspp(f, k, np.random.default_rng(child))
            assert np.array_equal(S[r], ref_cent), (n, r)
            ref_labels, ref_cost2, _, ref_it = O.lloyd(f, k, ref_cent, 100, 1e-6)
            assert its[r] == ref_it
            assert abs(cst[r] - ref_cost2) <= COST_TOL * ref_cost2
            assert O.adjusted_rand(lab[r], ref_labels) >= 0.999


@pytest.mark.parametrize("n,d,k", [(60000, 64, 48), (30000, 128, 100), (20000, 24, 40), (8000, 37, 50)])
def test_fp32_screen_same_labels_as_fp64(P, n, d, k):
    """The FP32 screen of the lane path (csc_kmeans_plan_set_screen) decides
    only rows whose FP64 argmin it provably knows: labels and cost equal the
    FP64-only plan bit for bit, and match the oracle."""
    from paper_1706_03591_b200 import _native
    from paper_1706_03591_b200._device import upload_block
    import importlib
    KM = importlib.import_module("paper_1706_03591_b200.kmeans")
    f = blobs(n, d, k, 1.2, seed=k)
    blk = upload_block(f)
    kids = np.random.SeedSequence(k).spawn(3)
    cfg = P.KmeansConfig(restarts=3, max_iters=40)
    la, ca = KM.run_restarts(blk, d, k, cfg, kids, fused=False)
    pool = KM._LLOYD_POOL
    assert pool.screen
    for lane in pool.lanes:
        _native.call("csc_kmeans_plan_set_screen", lane.plan, None, 0, None)
    try:
        lb, cb = KM.run_restarts(blk, d, k, cfg, kids, fused=False)
    finally:
        for lane in pool.lanes:
            _native.call("csc_kmeans_plan_set_screen", lane.plan, KM.ptr(pool.F32), pool.ld32, KM.ptr(pool.fn32))
    assert np.array_equal(la, lb)
    assert ca == cb
    ref_labels, _, ref_cost = O.kmeans(f, k, restarts=3, max_iters=40, tol=1e-6, seed=k)
    assert O.adjusted_rand(la, ref_labels) >= 0.999
    assert abs(np.sqrt(ca) - ref_cost) <= COST_TOL * ref_cost


@pytest.mark.parametrize("n,d,k,spread", [(60000, 64, 48, 1.2), (50000, 96, 64, 3.0), (20000, 24, 40, 2.0),
                                          (8000, 37, 50, 1.5), (40000, 96, 64, 6.0)])
def test_tensor_core_screen_same_labels(P, n, d, k, spread):
    """The tcgen05 (kind::tf32, 3xTF32) screen, the FP32 SIMT screen and the
    FP64-only plan give bit-identical labels and cost (the screens decide only
    rows their error bound proves); wide spreads put many rows near ties."""
    from paper_1706_03591_b200 import _native
    from paper_1706_03591_b200._device import upload_block
    import importlib
    KM = importlib.import_module("paper_1706_03591_b200.kmeans")
    assert _native.lib().csc_kmeans_screen_supported(d, k)
    f = blobs(n, d, k, spread, seed=d + k)
    blk = upload_block(f)
    kids = np.random.SeedSequence(d).spawn(2)
    cfg = P.KmeansConfig(restarts=2, max_iters=30)
    out = {}
    try:
        for mode in ("tc", "simt", "fp64"):
            _native.call("csc_kmeans_tuning", b"screen_tc", 1 if mode == "tc" else 0)
            KM.run_restarts(blk, d, k, cfg, kids, fused=False)  # builds the pool for this shape
            pool = KM._LLOYD_POOL
            for lane in pool.lanes:
                if mode == "fp64":
                    _native.call("csc_kmeans_plan_set_screen", lane.plan, None, 0, None)
                else:
                    _native.call("csc_kmeans_plan_set_screen", lane.plan, KM.ptr(pool.F32), pool.ld32,
                                 KM.ptr(pool.fn32))
            out[mode] = KM.run_restarts(blk, d, k, cfg, kids, fused=False)
    finally:
        _native.call("csc_kmeans_tuning", b"screen_tc", 1)
        pool = KM._LLOYD_POOL
        for lane in pool.lanes:
            _native.call("csc_kmeans_plan_set_screen", lane.plan, KM.ptr(pool.F32), pool.ld32, KM.ptr(pool.fn32))
    for mode in ("tc", "simt"):
        assert np.array_equal(out[mode][0], out["fp64"][0]), mode
        assert out[mode][1] == out["fp64"][1], mode


@pytest.mark.parametrize("n,d,k", [(600_000, 128, 100), (500_000, 96, 64), (300_000, 37, 50),
                                   (200_000, 160, 16), (100_000, 64, 128), (50_000, 1, 7), (70_000, 200, 33)])
def test_tensor_core_distances_many_tiles(P, n, d, k):
    """The tcgen05 screen's distances with tens of 128-row tiles per CTA (the
    shared-memory ring wraps many times; d = 128, k = 100 has an odd ring depth):
    every E within the stated bound of the exact fp64 distances, and five
    repeated calls bitwise equal (a pipeline race would show as a difference)."""
    import torch
    from paper_1706_03591_b200 import _native
    from paper_1706_03591_b200._device import ptr, stream
    if not _native.lib().csc_kmeans_tc_supported(d, k):
        pytest.skip(f"(d={d}, k={k}) outside the tensor-core screen")
    g = torch.Generator(device="cuda").manual_seed(n + d)
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
    outs = []
    for _ in range(5):
        E = torch.full((n, npad), float("nan"), dtype=torch.float32, device="cuda")
        _native.call("csc_kmeans_tc_distances", ptr(f32), n, d, ld32, ptr(fn32), ptr(c64), k, d, ptr(cnorm),
                     ptr(E), stream())
        outs.append(E)
    torch.cuda.synchronize()
    for E in outs[1:]:
        assert torch.equal(E, outs[0])
    D = (f64 ** 2).sum(1, keepdim=True) - 2 * f64 @ c64.T + cnorm[None, :]
    scale = (f64.norm(dim=1, keepdim=True) + cnorm.sqrt().max()) ** 2
    err = ((outs[0][:, :k].double() - D).abs() / scale).max().item()
    assert err <= (3 * d + 8) * 2.0 ** -23, err


@pytest.mark.parametrize("n,d,k,spread", [(400_000, 128, 100, 1.5), (300_000, 96, 64, 3.0)])
def test_tensor_core_screen_many_tiles_same_labels(P, n, d, k, spread):
    """As test_tensor_core_screen_same_labels, at sizes where every CTA of the
    persistent screen runs many tiles (the cfg3 / cfg5 regime)."""
    from paper_1706_03591_b200 import _native
    from paper_1706_03591_b200._device import upload_block
    import importlib
    KM = importlib.import_module("paper_1706_03591_b200.kmeans")
    f = blobs(n, d, k, spread, seed=n + k)
    blk = upload_block(f)
    kids = np.random.SeedSequence(n).spawn(1)
    cfg = P.KmeansConfig(restarts=1, max_iters=8)
    out = {}
    try:
        for mode in ("tc", "fp64"):
            _native.call("csc_kmeans_tuning", b"screen_tc", 1 if mode == "tc" else 0)
            KM.run_restarts(blk, d, k, cfg, kids, fused=False)
            pool = KM._LLOYD_POOL
            for lane in pool.lanes:
                if mode == "fp64":
                    _native.call("csc_kmeans_plan_set_screen", lane.plan, None, 0, None)
                else:
                    _native.call("csc_kmeans_plan_set_screen", lane.plan, KM.ptr(pool.F32), pool.ld32,
                                 KM.ptr(pool.fn32))
            out[mode] = KM.run_restarts(blk, d, k, cfg, kids, fused=False)
    finally:
        _native.call("csc_kmeans_tuning", b"screen_tc", 1)
        pool = KM._LLOYD_POOL
        for lane in pool.lanes:
            _native.call("csc_kmeans_plan_set_screen", lane.plan, KM.ptr(pool.F32), pool.ld32, KM.ptr(pool.fn32))
    assert np.array_equal(out["tc"][0], out["fp64"][0])
    assert out["tc"][1] == out["fp64"][1]


@pytest.mark.parametrize("n,d,k", [(200_000, 96, 64), (60_000, 128, 100), (30_000, 17, 5)])
def test_exact_sums_match_row_order_sums(P, n, d, k):
    """The Lloyd plan's exact fixed-point centroid sums (changed rows only,
    order-free) against the row-ordered per-chunk sums: same labels, cost to
    1e-12 relative, both within the oracle's tolerances."""
    from paper_1706_03591_b200 import _native
    from paper_1706_03591_b200._device import upload_block
    import importlib
    KM = importlib.import_module("paper_1706_03591_b200.kmeans")
    f = blobs(n, d, k, 1.5, seed=n + d)
    blk = upload_block(f)
    kids = np.random.SeedSequence(d + k).spawn(2)
    cfg = P.KmeansConfig(restarts=2, max_iters=30)
    out = {}
    try:
        for exact in (1, 0):
            _native.call("csc_kmeans_tuning", b"update_exact", exact)
            KM._LLOYD_POOLS.clear()  # plans read the knob when they are created
            out[exact] = KM.run_restarts(blk, d, k, cfg, kids, fused=False)
    finally:
        _native.call("csc_kmeans_tuning", b"update_exact", 1)
        KM._LLOYD_POOLS.clear()
    assert np.array_equal(out[1][0], out[0][0])
    assert abs(out[1][1] - out[0][1]) <= 1e-12 * out[0][1]
    ref_labels, _, ref_cost = O.kmeans(f, k, restarts=2, max_iters=30, tol=1e-6, seed=d + k)
    assert O.adjusted_rand(out[1][0], ref_labels) >= 0.999
    assert abs(np.sqrt(out[1][1]) - ref_cost) <= COST_TOL * ref_cost


@pytest.mark.parametrize("screen", ["tc", "fp64"])
def test_plan_empty_cluster_repair_exact_sums(P, screen):
    """The Lloyd plan (csc_kmeans_iterate: screened assignment, exact
    fixed-point sums updated from the changed rows) through the empty-cluster
    repair (kmeans.py:99-108): seeds far from every row leave clusters empty
    on the first assignment and the reseeded rows move between clusters;
    labels equal the oracle's Lloyd from the same seeds exactly, iterations
    and cost agree."""
    import importlib
    import torch
    from paper_1706_03591_b200 import _native
    from paper_1706_03591_b200._device import ptr, upload_block
    KM = importlib.import_module("paper_1706_03591_b200.kmeans")
    rng = np.random.default_rng(11)
    n, d, k = 6000, 64, 16  # inside the tensor-core screen's shapes
    f = rng.normal(size=(n, d)) + 4.0 * rng.integers(0, 4, size=(n, 1))
    c0 = f[rng.choice(n, k, replace=False)].copy()
    for j in (2, 9, 13):
        c0[j] = 1e3 + 10.0 * j
    blk = upload_block(f)
    ws = KM._Workspace(blk, d, k)
    plan = ws._plan()
    if screen == "tc":
        ld32 = (d + 3) // 4 * 4
        f32 = torch.zeros((n, ld32), dtype=torch.float32, device=blk.device)
        fn32 = torch.empty(n, dtype=torch.float32, device=blk.device)
        _native.call("csc_kmeans_screen_prepare", ptr(blk), n, d, blk.shape[1], ptr(f32), ld32, ptr(fn32),
                     KM.stream())
        _native.call("csc_kmeans_plan_set_screen", plan, ptr(f32), ld32, ptr(fn32))
    ws.cent[:, :d].copy_(torch.from_numpy(c0))
    hist = []
    cost2 = ws.lloyd(100, 1e-6, history=hist)
    labels = ws.labels.cpu().numpy().astype(np.int64)
    ref_labels, ref_cost2, _, ref_it = O.lloyd(f, k, c0, 100, 1e-6)
    assert len(hist) == ref_it
    assert np.array_equal(labels, ref_labels)
    assert abs(cost2 - ref_cost2) <= COST_TOL * ref_cost2


@pytest.mark.parametrize("n,d,k,R", [(300_000, 37, 6, 3), (600_000, 96, 5, 10), (270_001, 16, 4, 2),
                                     (263_000, 130, 3, 7)])
def test_batched_kpp_staged_equals_direct_and_reference(P, n, d, k, R):
    """csc_kmeanspp_batch's shared-memory-staged distance pass (rows >= 256 per
    chunk, 16-byte-aligned block) gives bitwise the seeds of the direct pass,
    and both pick the reference's rows (kmeans.py:64-77)."""
    from paper_1706_03591_b200 import _native
    from paper_1706_03591_b200._device import upload_block
    from paper_1706_03591_b200.kmeans import _Workspace, batched_kmeanspp
    f = blobs(n, d, max(k, 8), 1.5, 5)
    ws = _Workspace(upload_block(f), d, k)
    kids = np.random.SeedSequence(11).spawn(R)
    try:
        _native.call("csc_kmeans_tuning", b"kpp_staged", 1)
        staged = batched_kmeanspp(ws, kids).cpu().numpy()
        _native.call("csc_kmeans_tuning", b"kpp_staged", 0)
        direct = batched_kmeanspp(ws, kids).cpu().numpy()
    finally:
        _native.call("csc_kmeans_tuning", b"kpp_staged", 1)
    assert np.array_equal(staged, direct)
    for r in range(min(R, 2)):
        ref, _ = O.kmeanspp(f, k, np.random.default_rng(kids[r]))
        assert np.array_equal(staged[r, :, :d], ref), r
