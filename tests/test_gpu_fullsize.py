"""GPU checks at BASELINE's full sizes through size-independent properties.

cfg3 scale (n = 1M planted partition, nnz(L) = 33M): the CPU oracle cannot run
the whole path here in seconds, so these compare sampled rows against CPU
arithmetic and check identities that hold at any size:
  * Laplacian rows bit-exact on a row sample (graphs.py:349-361 recipe) and
    L D^(1/2) 1 = 0;
  * filter linearity, column-split invariance (bitwise), first order vs CPU;
  * moment energy == ||filtered||^2 (the single-pass bisection's identity);
  * k-means assignment == exact argmin on a row sample;
  * edge deltas == numpy set algebra (bitwise codes).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, K, DEG, RATIO = 1_000_000, 100, 32.0, 0.02


@pytest.fixture(scope="module")
def big(cuda_ok):
    import paper_1706_03591_b200 as P
    from paper_1706_03591_b200 import generators as G
    q1, q2 = G.sbm_probabilities(N, K, DEG, RATIO)
    codes = G.planted_partition_codes(N, K, q1, q2, 3)
    g = G.graph_from_codes(N, codes)
    lap = P.laplacian(g)
    return P, G, codes, g, lap, (q1, q2)


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def test_fullsize_laplacian_rows_bitwise_and_null_vector(big):
    P, G, codes, g, lap, _ = big
    m = lap.matrix
    lo, hi = codes // N, codes % N
    deg = (np.bincount(lo, minlength=N) + np.bincount(hi, minlength=N)).astype(np.float64)
    inv = np.zeros(N)
    nz = deg > 0
    inv[nz] = 1.0 / np.sqrt(deg[nz])
    order_hi = np.argsort(hi, kind="stable")
    hi_sorted = hi[order_hi]
    rng = np.random.default_rng(0)
    for i in rng.choice(N, 2000, replace=False):
        a0, a1 = np.searchsorted(lo, [i, i + 1])
        b0, b1 = np.searchsorted(hi_sorted, [i, i + 1])
        nbr = np.sort(np.concatenate([hi[a0:a1], lo[order_hi[b0:b1]]]))
        cols = np.sort(np.concatenate([nbr, [i]])) if deg[i] > 0 else np.array([], np.int64)
        vals = np.where(cols == i, 1.0, -((inv[i] * 1.0) * inv[cols]))
        s, e = m.indptr[i], m.indptr[i + 1]
        assert np.array_equal(m.indices[s:e], cols)
        assert np.array_equal(m.data[s:e], vals)
    assert m.nnz == 2 * codes.size + int(nz.sum())
    r = m @ np.sqrt(deg)
    assert np.abs(r).max() <= 1e-12 * np.sqrt(deg).max()


def test_fullsize_filter_linearity_columns_and_first_order(big):
    import torch
    from paper_1706_03591_b200.filters import filter_block
    from paper_1706_03591_b200.signals import device_signals
    P, G, codes, g, lap, _ = big
    d = 16
    x = device_signals(N, d, 1)
    y = device_signals(N, d, 2)
    poly = P.cheb_coeffs(0.6, lap.lambda_max_bound, 20)
    fx, _ = filter_block(lap, poly, x, d)
    fy, _ = filter_block(lap, poly, y, d)
    fxy, _ = filter_block(lap, poly, 0.75 * x - 1.5 * y, d)
    assert _rel(fxy.cpu(), (0.75 * fx - 1.5 * fy).cpu()) <= 1e-12
    # columns are independent recurrences: a column slice filtered alone is bitwise the same
    half = torch.zeros_like(x)
    half[:, :8] = x[:, :8]
    fh, _ = filter_block(lap, poly, half, 8)
    assert torch.equal(fh[:, :8], fx[:, :8])
    # first order (coefficients 0, 1 -> out = M x, M = I - (2/lambda_max) L) on sampled rows
    one = P.FilterPoly(1, np.array([0.0, 1.0]), 0.0, lap.lambda_max_bound, "")
    t1, _ = filter_block(lap, one, x, d)
    m = lap.matrix
    s = 2.0 / lap.lambda_max_bound
    xh = x[:, :d].cpu().numpy()
    t1h = t1[:, :d].cpu().numpy()
    rng = np.random.default_rng(1)
    for i in rng.choice(N, 500, replace=False):
        a, b = m.indptr[i], m.indptr[i + 1]
        cols, vals = m.indices[a:b], m.data[a:b]
        mv = np.where(cols == i, 1.0 - s * vals, -s * vals)
        ref = mv @ xh[cols]
        assert np.abs(t1h[i] - ref).max() <= 1e-13 * max(np.abs(ref).max(), 1.0)


def test_fullsize_moment_energy_identity(big):
    from paper_1706_03591_b200.filters import MOMENT_GUARD, block_moments, filter_block, moment_energy
    from paper_1706_03591_b200.signals import device_signals
    P, G, codes, g, lap, _ = big
    d, m = 8, 30
    x = device_signals(N, d, 5)
    mu = block_moments(lap, x, d, m, lap.lambda_max_bound)
    assert abs(mu[0] - float((x[:, :d] ** 2).sum().item())) <= 1e-12 * mu[0]
    for cut in (0.1, 0.6, 1.4):
        poly = P.cheb_coeffs(cut, lap.lambda_max_bound, m)
        _, s = filter_block(lap, poly, x, d, want_sumsq=True)
        e = float(s.item())
        # the moment form cancels ~1e6-sized terms down to the energy: at this size
        # its error (~5e-11 at low cutoffs) must stay well inside the bisection's
        # guard band (MOMENT_GUARD * k count units), where decisions are re-checked
        assert abs(moment_energy(mu, poly.coeffs) - e) <= 0.1 * MOMENT_GUARD * max(e, 1.0)


def test_fullsize_kmeans_assignment_is_exact_argmin(big):
    import torch
    from paper_1706_03591_b200 import _native
    from paper_1706_03591_b200._device import ptr, row_stride, stream
    P, G, codes, g, lap, _ = big
    d, k = 24, 100
    gen = torch.Generator(device="cuda").manual_seed(7)
    ld = row_stride(d)
    f = torch.zeros((N, ld), dtype=torch.float64, device="cuda")
    f[:, :d] = torch.randn((N, d), dtype=torch.float64, device="cuda", generator=gen)
    c = torch.zeros((k, ld), dtype=torch.float64, device="cuda")
    c[:, :d] = torch.randn((k, d), dtype=torch.float64, device="cuda", generator=gen)
    fn = torch.empty(N, dtype=torch.float64, device="cuda")
    cn = torch.empty(k, dtype=torch.float64, device="cuda")
    _native.call("csc_kmeans_rownorms", ptr(f), N, d, ld, ptr(fn), stream())
    _native.call("csc_kmeans_rownorms", ptr(c), k, d, ld, ptr(cn), stream())
    labels = torch.empty(N, dtype=torch.int32, device="cuda")
    own = torch.empty(N, dtype=torch.float64, device="cuda")
    counts = torch.empty(k, dtype=torch.int32, device="cuda")
    _native.call("csc_kmeans_assign", ptr(f), ptr(fn), N, d, ld, ptr(c), ld, ptr(cn), k, ptr(labels), ptr(own),
                 ptr(counts), stream())
    lab = labels.cpu().numpy()
    assert int(counts.sum().item()) == N
    assert np.array_equal(np.bincount(lab, minlength=k), counts.cpu().numpy())
    fh, ch = f[:, :d].cpu().numpy(), c[:, :d].cpu().numpy()
    rows = np.random.default_rng(3).choice(N, 5000, replace=False)
    d2 = ((fh[rows, None, :] - ch[None, :, :]) ** 2).sum(-1)
    srt = np.sort(d2, axis=1)
    clear = (srt[:, 1] - srt[:, 0]) > 1e-9 * (1.0 + srt[:, 0])  # not a rounding-level near-tie
    assert clear.mean() > 0.99
    assert np.array_equal(lab[rows][clear], d2.argmin(1)[clear])


def test_fullsize_edge_delta_codes(big):
    P, G, codes, g, lap, (q1, q2) = big
    labels = np.repeat(np.arange(K), G.block_sizes(N, K))
    dl, il = G.edge_churn(codes, N, labels, q1, q2, 0.01, seed=9)
    g2 = g.apply_delta(dl, il)
    expect = np.union1d(np.setdiff1d(codes, dl, assume_unique=True), il)
    assert np.array_equal(g2.edge_codes(), expect)
    lap2 = P.laplacian(g2)
    assert lap2.matrix.nnz == 2 * expect.size + int(np.count_nonzero(
        np.bincount(expect // N, minlength=N) + np.bincount(expect % N, minlength=N)))
