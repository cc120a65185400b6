"""GPU parity: libcscb200 through the drop-in API vs the pinned CPU oracle.

Tolerances (north_star): Laplacian / CSR updates bit-exact; fp64 features
relative Frobenius <= 1e-10; lambda_k in the same bisection interval (here:
identical probe sequence); k-means from the reference's initial centroids
ARI >= 0.999 and cost within 1e-9 relative. fp32 is reported separately
(<= 1e-4 here, measured values in DESIGN.md).
"""
import numpy as np
import pytest

from conftest import golden
from oracle import csc_oracle as O
from oracle import native as ON

pytestmark = pytest.mark.gpu

FEAT_TOL = 1e-10


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def P(cuda_ok):
    import paper_1706_03591_b200 as P
    return P


def graph_from(g, name, P):
    return P.Graph(int(g[f"{name}_n"]), g[f"{name}_i"], g[f"{name}_j"], g[f"{name}_w"])


# ---------------------------------------------------------------------------
# Laplacian: bit-exact (graphs.py:339-362)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["path3", "path10", "triangle", "isolated", "single", "empty",
                                  "sbm60", "weighted"])
@pytest.mark.parametrize("variant", ["normalized", "combinatorial"])
def test_laplacian_bitwise_small(P, name, variant):
    g = golden("small")
    lap = P.laplacian(graph_from(g, name, P), variant)
    m = lap.matrix
    p = f"{name}_{variant}"
    assert np.array_equal(m.indptr, g[f"{p}_indptr"])
    assert np.array_equal(m.indices, g[f"{p}_indices"])
    assert np.array_equal(m.data, g[f"{p}_data"])
    assert lap.lambda_max_bound == float(g[f"{p}_bound"])


def test_laplacian_bitwise_cfg1(P):
    g = golden("cfg1")
    lap = P.laplacian(graph_from(g, "g", P))
    m = lap.matrix
    assert np.array_equal(m.indptr, g["L_indptr"])
    assert np.array_equal(m.indices, g["L_indices"])
    assert np.array_equal(m.data, g["L_data"])


def test_laplacian_random_weighted_bitwise(P):
    rng = np.random.default_rng(3)
    n = 3000
    m = 40000
    i = rng.integers(0, n, m)
    j = rng.integers(0, n, m)
    ok = i != j
    code = np.unique(np.minimum(i, j)[ok] * n + np.maximum(i, j)[ok])
    lo, hi = code // n, code % n
    w = rng.uniform(0.01, 5.0, code.size)
    perm = rng.permutation(code.size)
    g = P.Graph(n, hi[perm], lo[perm], w[perm])
    for variant in ("normalized", "combinatorial"):
        lap = P.laplacian(g, variant)
        ip, ix, dv, bound = O.laplacian_csr(n, g.edge_i, g.edge_j, g.edge_w, variant)
        assert np.array_equal(lap.matrix.indptr, ip)
        assert np.array_equal(lap.matrix.indices, ix)
        assert np.array_equal(lap.matrix.data, dv)
        assert lap.lambda_max_bound == bound


# ---------------------------------------------------------------------------
# Filter (filters.py:155-187)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("tag", ["m37", "m40none", "sig60", "ident", "lin", "allpass"])
def test_filter_small_golden(P, tag):
    g = golden("small")
    lap = P.laplacian(graph_from(g, "sbm60", P))
    poly = P.FilterPoly(len(g[f"f60_{tag}_coeffs"]) - 1, g[f"f60_{tag}_coeffs"], 1.0,
                        float(g[f"f60_{tag}_lmax"]), "none")
    counter = P.MatvecCounter()
    out = P.apply_filter(lap, poly, g["f60_x"], counter)
    assert rel(out, g[f"f60_{tag}_out"]) <= FEAT_TOL
    assert counter.count == (len(poly.coeffs) - 1) * 6


def test_filter_identity_and_linear_kats(P):
    g = golden("small")
    lap = P.laplacian(graph_from(g, "sbm60", P))
    x = np.random.default_rng(0).normal(size=(lap.n, 4))
    ident = P.FilterPoly(5, np.array([1.0, 0, 0, 0, 0, 0]), 1.0, 2.0, "none")
    assert np.allclose(P.apply_filter(lap, ident, x), x, atol=1e-14)
    lmax = lap.lambda_max_bound
    lin = P.FilterPoly(1, np.array([lmax / 2, -lmax / 2]), 1.0, lmax, "none")
    x3 = np.random.default_rng(1).normal(size=(lap.n, 3))
    assert np.allclose(P.apply_filter(lap, lin, x3), lap.matrix @ x3, atol=1e-10)


def test_filter_cfg1_golden_and_fp32(P):
    g = golden("cfg1")
    lap = P.laplacian(graph_from(g, "g", P))
    poly = P.cheb_coeffs(0.5, 2.0, 50)
    assert np.array_equal(poly.coeffs, g["coeffs_05"])
    out = P.apply_filter(lap, poly, g["R"])
    assert rel(out, g["filt_05"]) <= FEAT_TOL
    out32 = P.apply_filter(lap, poly, g["R"], precision="fp32")
    e32 = rel(out32, g["filt_05"])
    print(f"cfg1 fp32 rel Frobenius error {e32:.3e}")
    assert e32 <= 1e-4


def test_filter_combinatorial_weighted(P):
    g = golden("small")
    lap = P.laplacian(graph_from(g, "weighted", P), "combinatorial")
    poly = P.FilterPoly(30, g["fw_coeffs"], 1.0, float(g["fw_lmax"]), "jackson")
    out = P.apply_filter(lap, poly, g["fw_x"])
    assert rel(out, g["fw_out"]) <= FEAT_TOL


@pytest.mark.parametrize("d", [1, 2, 3, 5, 8, 17, 40, 64, 100, 128, 200, 600])
def test_filter_widths(P, d):
    """Every row-group/vector template and the >256-vector column chunking."""
    g = golden("cfg1")
    lap = P.laplacian(graph_from(g, "g", P))
    x = np.random.default_rng(d).normal(size=(lap.n, d))
    poly = P.cheb_coeffs(0.7, 2.0, 12)
    out = P.apply_filter(lap, poly, x)
    ref = ON.cheb_filter(g["L_indptr"], g["L_indices"], g["L_data"], 2.0, poly.coeffs, x)
    assert rel(out, ref) <= FEAT_TOL


def test_filter_long_rows_segment_path(P):
    """Hub rows above the long-row threshold go through the segment kernels."""
    rng = np.random.default_rng(7)
    n = 6000
    hubs = [0, 17, 4000]
    ii, jj = [], []
    for h, deg in zip(hubs, [5000, 2500, 1100]):
        nb = rng.choice(np.setdiff1d(np.arange(n), [h]), size=deg, replace=False)
        ii.append(np.full(deg, h))
        jj.append(nb)
    base_i = rng.integers(0, n, 30000)
    base_j = rng.integers(0, n, 30000)
    ii.append(base_i)
    jj.append(base_j)
    i = np.concatenate(ii)
    j = np.concatenate(jj)
    ok = i != j
    code = np.unique(np.minimum(i, j)[ok] * n + np.maximum(i, j)[ok])
    g = P.Graph(n, code // n, code % n, np.ones(code.size))
    lap = P.laplacian(g)
    plan = lap.plan(1.0)
    assert plan.n_long >= 3 and plan.n_seg > plan.n_long
    for d in (3, 40, 128):
        x = rng.normal(size=(n, d))
        poly = P.cheb_coeffs(0.4, 2.0, 20)
        out = P.apply_filter(lap, poly, x)
        m = lap.matrix
        ref = ON.cheb_filter(m.indptr, m.indices, m.data, 2.0, poly.coeffs, x)
        assert rel(out, ref) <= FEAT_TOL
        est, _ = P.eigencount(lap, 0.4, d, m=20, seed=1)
        r = O.random_signals(n, d, 1)
        ref_e = float((ON.cheb_filter(m.indptr, m.indices, m.data, 2.0, poly.coeffs, r) ** 2).sum())
        assert abs(est - ref_e) <= 1e-10 * ref_e


def test_filter_deterministic(P):
    g = golden("cfg1")
    lap = P.laplacian(graph_from(g, "g", P))
    poly = P.cheb_coeffs(0.5, 2.0, 50)
    a = P.apply_filter(lap, poly, g["R"])
    b = P.apply_filter(lap, poly, g["R"])
    assert np.array_equal(a, b)


def test_filter_errors(P):
    g = golden("small")
    lap = P.laplacian(graph_from(g, "sbm60", P))
    poly = P.cheb_coeffs(0.5, 2.0, 5)
    with pytest.raises(ValueError):
        P.apply_filter(lap, poly, np.zeros(lap.n))
    with pytest.raises(ValueError):
        P.apply_filter(lap, poly, np.zeros((lap.n + 1, 2)))


def test_filter_from_scipy_laplacian(P):
    """A user-built LaplacianMatrix (SciPy CSR) is uploaded on first use."""
    import scipy.sparse as sp
    g = golden("cfg1")
    mat = sp.csr_matrix((g["L_data"], g["L_indices"], g["L_indptr"]), shape=(1000, 1000))
    lap = P.LaplacianMatrix(mat, "normalized", 2.0)
    out = P.apply_filter(lap, P.FilterPoly(50, g["coeffs_05"], 0.5, 2.0, "jackson"), g["R"])
    assert rel(out, g["filt_05"]) <= FEAT_TOL


# ---------------------------------------------------------------------------
# Eigencount bisection (filters.py:199-277)
# ---------------------------------------------------------------------------

def test_bisection_cfg1_same_probes(P):
    g = golden("cfg1")
    lap = P.laplacian(graph_from(g, "g", P))
    from paper_1706_03591_b200.filters import _search_cutoff
    counter = P.MatvecCounter()
    cfg = P.FilterConfig(order=50, max_iters=8)
    cut, filt, poly, iters, est = _search_cutoff(lap, 10, g["R"], (0.0, 2.0), cfg, counter, 1.0)
    assert cut == float(g["cutoff"]) and iters == int(g["iters"])
    assert abs(est - float(g["est"])) <= 1e-10 * float(g["est"])
    assert rel(filt, g["features"]) <= FEAT_TOL
    assert counter.count == iters * 50 * 40


def test_find_lambda_k_small_trace(P):
    g = golden("small")
    lap = P.laplacian(graph_from(g, "sbm60", P))
    counter = P.MatvecCounter()
    lam, feats, iters = P.find_lambda_k(lap, 3, d=12, m=40, seed=5, counter=counter)
    assert lam == float(g["flk_lambda"]) and iters == int(g["flk_iters"])
    assert rel(feats.values, g["flk_features"]) <= FEAT_TOL
    assert counter.count == iters * 40 * 12


def test_search_errors(P):
    g = golden("small")
    lap = P.laplacian(graph_from(g, "sbm60", P))
    with pytest.raises(ValueError):
        P.find_lambda_k(lap, 3, d=10, interval=(1.0, 0.5))
    with pytest.raises(ValueError):
        P.find_lambda_k(lap, lap.n, d=10)
    # non-convergence carries the reference's error fields
    cl = P.Graph(10, *np.triu_indices(5, 1), np.ones(10))
    lap2 = P.laplacian(cl)
    with pytest.raises(P.EigencountSearchError) as err:
        P.find_lambda_k(lap2, 2, d=100, m=60, seed=6, interval=(1.9, 2.0), tol=0.0, max_iters=2)
    assert err.value.iterations == 2
    assert 1.9 < err.value.last_cutoff < 2.0


# ---------------------------------------------------------------------------
# k-means (kmeans.py)
# ---------------------------------------------------------------------------

def test_kmeanspp_same_picks_and_lloyd_from_reference_init(P):
    g = golden("cfg1")
    f = g["features"]
    from paper_1706_03591_b200.kmeans import _Workspace
    from paper_1706_03591_b200._device import upload_block
    import torch
    blk = upload_block(f)
    ws = _Workspace(blk, 40, 10)
    child = np.random.SeedSequence(0).spawn(2)[1].spawn(1)[0]
    picks = []
    ws.kmeanspp(np.random.default_rng(child), record=picks)
    _, ref_picks = O.kmeanspp(f, 10, np.random.default_rng(child))
    assert picks == ref_picks
    cent = ws.cent[:, :40].cpu().numpy()
    assert np.array_equal(cent, g["km_init"])
    hist = []
    cost2 = ws.lloyd(20, 1e-6, hist)
    labels = ws.labels.cpu().numpy()
    assert O.adjusted_rand(labels, g["km_labels"]) >= 0.999
    assert abs(cost2 - float(g["km_cost2"])) <= 1e-9 * float(g["km_cost2"])
    np.testing.assert_allclose(hist, g["km_hist"], rtol=1e-9)
    torch.cuda.synchronize()


def test_kmeans_goldens(P):
    g = golden("kmeans")
    a = P.kmeans(g["a_f"], 3, seed=123)
    assert O.adjusted_rand(a.labels, g["a_labels"]) >= 0.999
    assert abs(a.feature_cost - float(g["a_cost"])) <= 1e-9 * float(g["a_cost"])
    for s in range(6):
        b = P.kmeans(np.array([[0.0], [0.0], [5.0]]), 3, P.KmeansConfig(restarts=1), seed=s)
        assert np.array_equal(b.labels, g[f"dup{s}_labels"])
        assert b.cluster_sizes.min() >= 1
    r = P.kmeans(np.array([[0.0, 0.0], [2.0, 0.0], [0.0, 0.1], [2.0, 0.1]]), 2,
                 P.KmeansConfig(restarts=10), seed=0)
    assert np.isclose(r.feature_cost, float(g["rect_cost"]), rtol=1e-9)
    kb = P.kmeans(g["b_f"], 12, P.KmeansConfig(restarts=3, max_iters=50), seed=77)
    assert O.adjusted_rand(kb.labels, g["b_labels"]) >= 0.999
    assert abs(kb.feature_cost - float(g["b_cost"])) <= 1e-9 * float(g["b_cost"])


def test_kmeans_validation_and_cost(P):
    with pytest.raises(ValueError):
        P.kmeans(np.zeros((4, 2)), 5)
    with pytest.raises(ValueError):
        P.kmeans(np.zeros((4, 2)), 0)
    with pytest.raises(ValueError):
        P.kmeans(np.array([[np.nan, 0.0]]), 1)
    rng = np.random.default_rng(3)
    f = rng.normal(size=(30, 4))
    labels = rng.integers(0, 3, size=30)
    labels[:3] = [0, 1, 2]
    a = P.Assignment(labels, np.bincount(labels, minlength=3), 0.0)
    x = a.indicator()
    assert np.isclose(P.kmeans_cost(f, a), np.linalg.norm(f - x @ (x.T @ f)), atol=1e-10)
    six = P.kmeans(rng.normal(size=(6, 2)), 6, P.KmeansConfig(restarts=5), seed=1)
    assert six.cluster_sizes.tolist() == [1] * 6 and six.feature_cost <= 1e-12


# ---------------------------------------------------------------------------
# CSC + dynamic CSC end to end
# ---------------------------------------------------------------------------

def test_csc_assign_cfg1(P):
    g = golden("cfg1")
    lap = P.laplacian(graph_from(g, "g", P))
    counter = P.MatvecCounter()
    a, diag = P.csc_assign(lap, 10, 40, filter_cfg=P.FilterConfig(order=50, max_iters=8),
                           kmeans_cfg=P.KmeansConfig(restarts=1, max_iters=20), seed=0, counter=counter)
    assert diag.lambda_k == float(g["csc_lambda"]) and diag.search_iters == int(g["csc_iters"])
    assert diag.matvecs == int(g["csc_matvecs"]) == counter.count
    assert O.adjusted_rand(a.labels, g["csc_labels"]) >= 0.999
    assert abs(a.feature_cost - float(g["csc_cost"])) <= 1e-9 * float(g["csc_cost"])


def test_dynamic_sequence_small_golden(P):
    g = golden("dynamic_small")
    graphs = [graph_from(g, f"g{t}", P) for t in range(4)]
    cfg = P.DynamicConfig(k=4, d=40, p=0.5, filter=P.FilterConfig(order=60),
                          kmeans=P.KmeansConfig(restarts=6))
    a, state, diag = P.dynamic_init(graphs[0], cfg, seed=10)
    steps = [(a, state, diag)]
    for gt in graphs[1:]:
        a, state, diag = P.dynamic_step(state, gt, cfg)
        steps.append((a, state, diag))
    for t, (a, st, dg) in enumerate(steps):
        assert dg.lambda_k == float(g[f"s{t}_lambda"])
        assert dg.refined == bool(g[f"s{t}_refined"]) and dg.search_iters == int(g[f"s{t}_iters"])
        assert dg.reused == int(g[f"s{t}_reused"])
        assert dg.matvecs_total == int(g[f"s{t}_mv_total"]) and dg.matvecs_fresh == int(g[f"s{t}_mv_fresh"])
        assert np.array_equal(st.features.step_tags, g[f"s{t}_step_tags"])
        assert np.array_equal(st.features.stream_tags, g[f"s{t}_stream_tags"])
        assert rel(st.features.values, g[f"s{t}_features"]) <= FEAT_TOL
        assert O.adjusted_rand(a.labels, g[f"s{t}_labels"]) >= 0.999
        assert abs(a.feature_cost - float(g[f"s{t}_cost"])) <= 1e-9 * float(g[f"s{t}_cost"])


def test_dynamic_bitwise_reuse_and_refilter(P):
    g = golden("dynamic_small")
    g0, g1 = graph_from(g, "g0", P), graph_from(g, "g1", P)
    cfg = P.DynamicConfig(k=4, d=20, p=0.35, filter=P.FilterConfig(order=60),
                          kmeans=P.KmeansConfig(restarts=2))
    _, state, _ = P.dynamic_init(g0, cfg, seed=4)
    prev = state.features.values.copy()
    _, state2, diag = P.dynamic_step(state, g1, cfg)
    theta = state2.features
    assert diag.reused == 7
    for col in range(7):
        assert np.array_equal(theta.values[:, col], prev[:, int(theta.stream_tags[col])])
    # refined/fresh columns equal a direct apply_filter of the same raw draw
    ss = np.random.SeedSequence(4)
    ss.spawn(2)
    _, sig_ss, _ = ss.spawn(3)
    raw = P.random_signals(g1.n, 13, sig_ss, scale_dim=20)
    expected = P.apply_filter(P.laplacian(g1), state2.filter, raw)
    assert np.array_equal(theta.values[:, 7:], expected)


def test_edge_delta_matches_reference_sequence(P):
    """apply_delta on the GPU reproduces the reference's next graph and its Laplacian bit-exactly."""
    g = golden("dynamic_small")
    g0 = graph_from(g, "g0", P)
    for t in range(1, 4):
        nxt = graph_from(g, f"g{t}", P)
        prev_codes, next_codes = g0.edge_codes(), nxt.edge_codes()
        dl = np.setdiff1d(prev_codes, next_codes)
        il = np.setdiff1d(next_codes, prev_codes)
        gd = g0.apply_delta(dl, il)
        assert gd.m == nxt.m
        assert np.array_equal(gd.edge_codes(), next_codes)
        lap = P.laplacian(gd)
        ip, ix, dv, _ = O.laplacian_csr(nxt.n, nxt.edge_i, nxt.edge_j, nxt.edge_w)
        assert np.array_equal(lap.matrix.indptr, ip)
        assert np.array_equal(lap.matrix.indices, ix)
        assert np.array_equal(lap.matrix.data, dv)
        g0 = gd
    codes = g0.edge_codes()
    absent = next(c for c in range(1, g0.n) if c not in set(codes.tolist()))
    with pytest.raises(ValueError):
        g0.apply_delta([absent], [])       # deleting a non-edge
    with pytest.raises(ValueError):
        g0.apply_delta([], [codes[0]])     # inserting an existing edge


def _expected_M(m, s):
    """M = I - s L restated on the CPU: exact zeros dropped, isolated rows M_ii = 1."""
    import scipy.sparse as sp
    n = m.shape[0]
    rows, cols, vals = [], [], []
    for i in range(n):
        cs = m.indices[m.indptr[i]:m.indptr[i + 1]]
        vs = m.data[m.indptr[i]:m.indptr[i + 1]]
        lii = vs[cs == i][0] if np.any(cs == i) else 0.0
        ent = {int(c): -s * v for c, v in zip(cs, vs) if c != i}
        ent[i] = 1.0 - s * lii
        for c in sorted(ent):
            if ent[c] != 0.0:
                rows.append(i)
                cols.append(c)
                vals.append(ent[c])
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))


@pytest.mark.parametrize("name,variant", [("sbm60", "normalized"), ("weighted", "combinatorial"),
                                          ("weighted", "normalized"), ("isolated", "combinatorial")])
def test_operator_plan_bitwise(P, name, variant):
    from paper_1706_03591_b200.graphs import export_plan
    g = golden("small")
    lap = P.laplacian(graph_from(g, name, P), variant)
    s = 2.0 / lap.lambda_max_bound if lap.lambda_max_bound > 0 else 1.0
    ip, ix, vv, _, _ = export_plan(lap.plan(s))
    exp = _expected_M(lap.matrix, s)
    assert np.array_equal(ip, exp.indptr)
    assert np.array_equal(ix, exp.indices)
    assert np.array_equal(vv, exp.data)


# ---------------------------------------------------------------------------
# Chebyshev moments and the single-pass bisection
# ---------------------------------------------------------------------------

def _oracle_moments(m_csr, s, x, m):
    """mu_q = <x, T_q(M) x> (summed over columns) by the CPU recurrence."""
    import scipy.sparse as sp
    n = m_csr.shape[0]
    M = sp.identity(n) - s * m_csr
    t_prev, t_cur = x, M @ x
    mu = [float((x * x).sum()), float((x * t_cur).sum())]
    for _ in range(2, 2 * m + 1):
        t_prev, t_cur = t_cur, 2.0 * (M @ t_cur) - t_prev
        mu.append(float((x * t_cur).sum()))
    return np.array(mu)


@pytest.mark.parametrize("d", [5, 40, 600])
def test_moments_match_oracle(P, d):
    from paper_1706_03591_b200.filters import block_moments
    from paper_1706_03591_b200._device import upload_block
    g = golden("cfg1")
    lap = P.laplacian(graph_from(g, "g", P))
    x = np.random.default_rng(d).normal(size=(lap.n, d)) / np.sqrt(d)
    mu = block_moments(lap, upload_block(x), d, 30, 2.0)
    ref = _oracle_moments(lap.matrix, 1.0, x, 30)
    scale = np.abs(ref).max()
    assert np.abs(mu - ref).max() <= 1e-12 * scale


def test_moment_energy_equals_block_energy(P):
    from paper_1706_03591_b200.filters import block_moments, moment_energy
    from paper_1706_03591_b200._device import upload_block
    g = golden("cfg1")
    lap = P.laplacian(graph_from(g, "g", P))
    mu = block_moments(lap, upload_block(g["R"]), 40, 50, 2.0)
    for cut in (0.1, 0.3, 0.5, 1.0, 1.9):
        poly = P.cheb_coeffs(cut, 2.0, 50)
        ref = O.count_from_block(ON.cheb_filter(g["L_indptr"], g["L_indices"], g["L_data"], 2.0,
                                                poly.coeffs, g["R"]), 1.0)
        assert abs(moment_energy(mu, poly.coeffs) - ref) <= 1e-11 * max(ref, 1.0)


@pytest.mark.parametrize("keep", ["1", "0"])
@pytest.mark.parametrize("case", ["cfg1", "small"])
def test_moment_search_equals_probe_search(P, case, keep, monkeypatch):
    """Moment bisection == the reference's per-probe refiltering: same cutoff,
    probes and features bit for bit, with the orders resident in HBM (keep=1:
    exact features by csc_cheb_combine) or re-swept (keep=0)."""
    monkeypatch.setenv("CSC_KEEP_ORDERS", keep)
    from paper_1706_03591_b200.filters import _search_cutoff
    if case == "cfg1":
        g = golden("cfg1")
        lap = P.laplacian(graph_from(g, "g", P))
        r, k, order, iters_max = g["R"], 10, 50, 8
    else:
        g = golden("small")
        lap = P.laplacian(graph_from(g, "sbm60", P))
        r, k, order, iters_max = O.random_signals(60, 12, 5), 3, 40, 20
    res = {}
    for mode in ("moments", "probe"):
        cnt = P.MatvecCounter()
        cfg = P.FilterConfig(order=order, max_iters=iters_max, search=mode)
        res[mode] = (_search_cutoff(lap, k, r, (0.0, 2.0), cfg, cnt, 1.0), cnt)
    (cm, fm, pm, im, em), cntm = res["moments"]
    (cp, fp, pp, ip_, ep), cntp = res["probe"]
    assert cm == cp and im == ip_
    assert np.array_equal(fm, fp)
    assert abs(em - ep) <= 1e-12 * abs(ep)
    assert cntm.count == cntp.count == im * order * r.shape[1]
    if keep == "1":  # one sweep series in total
        assert cntm.physical == order * r.shape[1]
    else:  # moment pass + final features (+ guard-band confirmations)
        assert cntm.physical >= 2 * order * r.shape[1]


def test_reference_counter_accepted(P):
    """A counter without the physical ledger (like cscluster.MatvecCounter) works."""
    class RefCounter:
        def __init__(self):
            self.count = 0

        def add(self, k):
            self.count += int(k)
    g = golden("small")
    lap = P.laplacian(graph_from(g, "sbm60", P))
    c = RefCounter()
    lam, feats, iters = P.find_lambda_k(lap, 3, d=12, m=40, seed=5, counter=c)
    assert c.count == iters * 40 * 12


def test_refine_ledger_odd_width(P):
    """Stale cutoff -> refinement; ledger = order * n_fresh * (1 + iters) (test_dynamic.py:105-127)."""
    g = golden("dynamic_small")
    g0, g1 = graph_from(g, "g0", P), graph_from(g, "g1", P)
    cfg = P.DynamicConfig(k=4, d=26, p=0.5, filter=P.FilterConfig(order=60),
                          kmeans=P.KmeansConfig(restarts=2))
    _, state, _ = P.dynamic_init(g0, cfg, seed=6)
    state.lambda_k = 0.3
    state.filter = P.cheb_coeffs(0.15, 2.0, 60)
    _, state2, diag = P.dynamic_step(state, g1, cfg)
    assert diag.refined and diag.search_iters >= 1
    assert diag.matvecs_total == 60 * 13 * (1 + diag.search_iters)
    ss = np.random.SeedSequence(6)
    ss.spawn(2)
    _, sig_ss, _ = ss.spawn(3)
    raw = P.random_signals(g1.n, 13, sig_ss, scale_dim=26)
    poly = P.cheb_coeffs(state2.lambda_k, 2.0, 60)
    assert np.array_equal(state2.features.values[:, 13:], P.apply_filter(P.laplacian(g1), poly, raw))


def test_csc_features_small_d_ledger(P):
    g = golden("small")
    lap = P.laplacian(graph_from(g, "sbm60", P))
    c = P.MatvecCounter()
    with pytest.warns(UserWarning, match="rank-deficient"):
        feats, cut, poly = P.csc_features(lap, 3, 2, P.FilterConfig(order=30), seed=0, counter=c)
    assert feats.d == 2 and feats.values.shape == (60, 2)
    assert c.count % (30 * 2) == 0


def test_batched_kmeanspp_matches_sequential(P):
    """Batched seeding == per-restart sequential seeding == the reference picks."""
    from paper_1706_03591_b200.kmeans import _Workspace, batched_kmeanspp
    from paper_1706_03591_b200._device import upload_block
    g = golden("cfg1")
    f = g["features"]
    ws = _Workspace(upload_block(f), 40, 10)
    kids = np.random.SeedSequence(0).spawn(2)[1].spawn(5)
    seeds = batched_kmeanspp(ws, kids)
    for r, child in enumerate(kids):
        ref, _ = O.kmeanspp(f, 10, np.random.default_rng(child))
        assert np.array_equal(seeds[r, :, :40].cpu().numpy(), ref)
    # zero D^2 mass -> replay path (duplicate points; kmeans.py:70-72)
    dup = np.array([[0.0], [0.0], [5.0]])
    ws2 = _Workspace(upload_block(dup), 1, 3)
    kids2 = np.random.SeedSequence(3).spawn(4)
    seeds2 = batched_kmeanspp(ws2, kids2)
    for r, child in enumerate(kids2):
        ref, _ = O.kmeanspp(dup, 3, np.random.default_rng(child))
        assert np.array_equal(seeds2[r, :, :1].cpu().numpy(), ref)


def test_graph_lloyd_equals_host_driven(P):
    """csc_kmeans_run (device loop graph, concurrent lanes) == host-driven pruned Lloyd."""
    from paper_1706_03591_b200.kmeans import _Workspace, batched_kmeanspp, run_restarts
    from paper_1706_03591_b200._device import upload_block
    g = golden("kmeans")
    f = g["b_f"]
    blk = upload_block(f)
    kids = np.random.SeedSequence(77).spawn(3)
    cfg = P.KmeansConfig(restarts=3, max_iters=50)
    labels, cost2 = run_restarts(blk, 24, 12, cfg, kids, fused=False)
    ws = _Workspace(blk, 24, 12)
    seeds = batched_kmeanspp(ws, kids)
    best = None
    for r in range(3):
        ws.cent.copy_(seeds[r])
        c2 = ws.lloyd(50, 1e-6)
        if best is None or c2 < best[0]:
            best = (c2, ws.labels.cpu().numpy().astype(np.int64))
    assert np.array_equal(labels, best[1])
    assert cost2 == best[0]
    assert np.array_equal(labels, g["b_labels"])


def test_graph_small_canonical_order(P):
    """Small graphs are canonicalised on the device too (no host branch)."""
    g = P.Graph(4, [2, 0, 3], [0, 1, 1], [1.0, 2.0, 3.0])
    assert g._i is None  # built on the device
    assert g.edge_i.tolist() == [0, 0, 1] and g.edge_j.tolist() == [1, 2, 3]
    assert g.edge_w.tolist() == [2.0, 1.0, 3.0]
    assert g.m == 3 and np.array_equal(g.edge_codes(), [1, 2, 7])
    assert np.array_equal(g.degrees, [3.0, 5.0, 1.0, 3.0])
    for bad in [(4, [0], [0], [1.0]), (4, [0], [5], [1.0]), (4, [0], [1], [0.0]),
                (4, [0, 1], [1, 0], [1.0, 1.0]), (4, [0, 1], [1], [1.0]), (-1, [], [], [])]:
        with pytest.raises(ValueError):
            P.Graph(*bad)
    with pytest.raises(AttributeError):
        g.n = 5
    assert P.graphs_equal(g, P.Graph(4, [0, 2, 1], [1, 0, 3], [2.0, 1.0, 3.0]))
    e = P.Graph(5, [], [], [])
    assert e.m == 0 and P.laplacian(e).nnz == 0


def test_graph_device_canonicalisation(P):
    """K9 on device (graphs.py:29-54): same canonical order, weights and errors as the reference."""
    rng = np.random.default_rng(11)
    n = 50000
    m = 3 << 16
    a = rng.integers(0, n, m)
    b = rng.integers(0, n, m)
    ok = a != b
    code = np.unique(np.minimum(a, b)[ok] * n + np.maximum(a, b)[ok])
    lo, hi = code // n, code % n
    flip = rng.random(code.size) < 0.5
    ii, jj = np.where(flip, hi, lo), np.where(flip, lo, hi)
    perm = rng.permutation(code.size)
    ii, jj = ii[perm], jj[perm]
    w = rng.uniform(0.1, 2.0, code.size)
    g = P.Graph(n, ii, jj, w)
    assert g._i is None  # built on the device
    clo, chi, cw = O.canonical_edges(n, ii, jj, w)
    assert g.m == code.size
    assert np.array_equal(g.edge_i, clo) and np.array_equal(g.edge_j, chi) and np.array_equal(g.edge_w, cw)
    lap = P.laplacian(g)
    ip, ix, dv, _ = O.laplacian_csr(n, clo, chi, cw)
    assert np.array_equal(lap.matrix.indptr, ip) and np.array_equal(lap.matrix.data, dv)
    unit = P.Graph(n, ii, jj, np.ones(code.size))
    assert unit.unit_weights() and np.array_equal(unit.edge_codes(), code)
    bad_cases = [
        (np.r_[ii, n], np.r_[jj, 0], np.r_[w, 1.0], "out of range"),
        (np.r_[ii, 5], np.r_[jj, 5], np.r_[w, 1.0], "self-loops"),
        (ii, jj, np.r_[w[:-1], 0.0], "positive"),
        (np.r_[ii, jj[0]], np.r_[jj, ii[0]], np.r_[w, 1.0], "duplicate"),
    ]
    for bi, bj, bw, msg in bad_cases:
        with pytest.raises(ValueError, match=msg):
            P.Graph(n, bi, bj, bw)


@pytest.mark.parametrize("variant", ["normalized", "combinatorial"])
def test_operator_plan_long_rows_bitwise(P, variant):
    """Warp-built rows of M (> 32 entries) == the CPU restatement, bit for bit."""
    from paper_1706_03591_b200.graphs import export_plan
    rng = np.random.default_rng(21)
    n = 3000
    i = np.r_[np.zeros(2000, np.int64), np.full(700, 1500), rng.integers(0, n, 6000)]
    j = np.r_[rng.permutation(np.arange(1, n))[:2000], rng.permutation(np.arange(n))[:700],
              rng.integers(0, n, 6000)]
    ok = i != j
    code = np.unique(np.minimum(i, j)[ok] * n + np.maximum(i, j)[ok])
    w = rng.uniform(0.5, 2.0, code.size)
    g = P.Graph(n, code // n, code % n, w)
    lap = P.laplacian(g, variant)
    s = 2.0 / lap.lambda_max_bound
    ip, ix, vv, _, _ = export_plan(lap.plan(s))
    exp = _expected_M(lap.matrix, s)
    assert np.diff(lap.matrix.indptr).max() > 600
    assert np.array_equal(ip, exp.indptr)
    assert np.array_equal(ix, exp.indices)
    assert np.array_equal(vv, exp.data)
    x = rng.normal(size=(n, 6))
    poly = P.cheb_coeffs(0.3 * lap.lambda_max_bound, lap.lambda_max_bound, 15)
    m = lap.matrix
    ref = ON.cheb_filter(m.indptr, m.indices, m.data, lap.lambda_max_bound, poly.coeffs, x)
    assert rel(P.apply_filter(lap, poly, x), ref) <= FEAT_TOL


def test_dynamic_cfg2_golden(P):
    """BASELINE configs[1] (n=20k, k=20, d=80, p=0.5, m=60): init + 2 steps vs the live reference.

    The graph sequence is rebuilt with on-device edge deltas (the reference's
    perturbed_sequence, stored as delete/insert code lists).
    """
    g = golden("cfg2")
    g0 = graph_from(g, "g0", P)
    graphs = [g0]
    for t in (1, 2):
        graphs.append(graphs[-1].apply_delta(g[f"del{t}"], g[f"ins{t}"]))
    cfg = P.DynamicConfig(k=20, d=80, p=0.5, filter=P.FilterConfig(order=60))
    a, state, diag = P.dynamic_init(graphs[0], cfg, seed=0)
    results = [(a, state, diag)]
    for gt in graphs[1:]:
        a, state, diag = P.dynamic_step(state, gt, cfg)
        results.append((a, state, diag))
    rows = g["rows"]
    for t, (a, st, dg) in enumerate(results):
        assert dg.lambda_k == float(g[f"s{t}_lambda"])
        assert dg.search_iters == int(g[f"s{t}_iters"]) and dg.refined == bool(g[f"s{t}_refined"])
        assert dg.matvecs_total == int(g[f"s{t}_mv_total"])
        assert np.array_equal(st.features.step_tags, g[f"s{t}_step_tags"])
        assert np.array_equal(st.features.stream_tags, g[f"s{t}_stream_tags"])
        v = st.features.values
        assert rel((v ** 2).sum(axis=0), g[f"s{t}_colnorm2"]) <= FEAT_TOL
        assert rel(v[rows], g[f"s{t}_rowsample"]) <= FEAT_TOL
        ari = O.adjusted_rand(a.labels, g[f"s{t}_labels"].astype(np.int64))
        print(f"cfg2 step {t}: ARI {ari:.6f} cost {a.feature_cost:.12f} ref {float(g[f's{t}_cost']):.12f}")
        assert ari >= 0.999
        assert abs(a.feature_cost - float(g[f"s{t}_cost"])) <= 1e-9 * float(g[f"s{t}_cost"])


def test_combine_equals_filter_bitwise(P):
    """csc_cheb_combine over resident orders == csc_cheb_filter, bit for bit, and the
    kept moment pass returns the same moments as the ring-buffer pass."""
    import torch
    from paper_1706_03591_b200._device import upload_block
    from paper_1706_03591_b200.filters import block_moments, block_moments_keep, combine_orders, filter_block
    g = golden("cfg1")
    lap = P.laplacian(graph_from(g, "g", P))
    blk = upload_block(g["R"])
    n, ld = blk.shape
    m = 37
    keep = torch.empty((m, n, ld), dtype=torch.float64, device=blk.device)
    mu_keep = block_moments_keep(lap, blk, 40, m, 2.0, keep)
    mu = block_moments(lap, blk, 40, m, 2.0)
    assert np.array_equal(mu_keep, mu)
    for cut in (0.05, 0.4, 1.3):
        poly = P.cheb_coeffs(cut, 2.0, m)
        ref, s_ref = filter_block(lap, poly, blk, 40, want_sumsq=True)
        out, s = combine_orders(blk, keep, 40, poly.coeffs)
        assert torch.equal(out, ref)
        assert abs(float(s.item()) - float(s_ref.item())) <= 1e-13 * float(s_ref.item())


def test_kmeans_zero_mass_replay_through_restarts(P):
    """Duplicate points exhaust the D^2 mass during seeding (the reference then
    draws integers(n), kmeans.py:70-72): the deferred replay in run_restarts
    must give the oracle's labels and cost for every seed."""
    f = np.array([[0.0, 0.0], [0.0, 0.0], [5.0, 1.0], [5.0, 1.0], [0.0, 0.0], [9.0, -2.0]])
    for seed in range(6):
        cfg = P.KmeansConfig(restarts=4, max_iters=20)
        asg = P.kmeans(f, 3, cfg, seed=seed)
        ref_labels, _, ref_cost = O.kmeans(f, 3, restarts=4, max_iters=20, tol=1e-6, seed=seed)
        assert np.array_equal(asg.labels, ref_labels)
        assert abs(asg.feature_cost - ref_cost) <= 1e-12 * max(ref_cost, 1.0)


def test_filter_host_pipeline(P, monkeypatch):
    """apply_filter's pinned-host pipeline (column chunks, copies overlapped with
    the filter on a side stream) returns the device path's features and charges
    the same matvecs."""
    import torch
    from paper_1706_03591_b200 import filters as PF
    g = golden("cfg1")
    lap = P.laplacian(graph_from(g, "g", P))
    poly = P.cheb_coeffs(0.5, 2.0, 50)
    x = torch.from_numpy(np.ascontiguousarray(g["R"], dtype=np.float64)).pin_memory().numpy()
    monkeypatch.setattr(PF, "PIPE_MIN_BYTES", 0)
    monkeypatch.setattr(PF, "PIPE_MIN_COLS", 4)
    monkeypatch.setattr(PF, "PIPE_MODE", "columns")
    for chunks in (2, 3):
        monkeypatch.setattr(PF, "PIPE_CHUNKS", chunks)
        counter = P.MatvecCounter()
        out = P.apply_filter(lap, poly, x, counter)
        assert rel(out, g["filt_05"]) <= FEAT_TOL
        assert counter.count == 50 * x.shape[1]
    # row-slice pipeline (the default): pinned and pageable input, any slice count
    monkeypatch.setattr(PF, "PIPE_MODE", "slices")
    dev = P.apply_filter(lap, poly, torch.from_numpy(x).cuda()).cpu().numpy()
    for slices, up in ((1, 1), (3, 2), (8, 8), (999, 7)):
        monkeypatch.setattr(PF, "PIPE_SLICES", slices)
        monkeypatch.setattr(PF, "PIPE_UP_SLICES", up)
        for xin in (x, np.array(x)):  # pinned pages, then an ordinary array
            counter = P.MatvecCounter()
            out = P.apply_filter(lap, poly, xin, counter)
            assert np.array_equal(out, dev), (slices, up)
            assert rel(out, g["filt_05"]) <= FEAT_TOL
            assert counter.count == 50 * x.shape[1]
    one = P.apply_filter(lap, P.cheb_coeffs(0.5, 2.0, 1), x)  # the last order is the first
    assert np.array_equal(one, P.apply_filter(lap, P.cheb_coeffs(0.5, 2.0, 1), torch.from_numpy(x).cuda()).cpu().numpy())
    monkeypatch.setattr(PF, "PIPE_MODE", "columns")
    # a larger block: pipelined host result equals the device-tensor path
    rng = np.random.default_rng(7)
    n, d = 60000, 96
    a, b = rng.integers(0, n, 8 * n), rng.integers(0, n, 8 * n)
    pairs = np.unique(np.stack([np.minimum(a, b), np.maximum(a, b)], 1)[a != b], axis=0)
    big = P.laplacian(P.Graph(n, pairs[:, 0], pairs[:, 1], rng.uniform(0.5, 2.0, len(pairs))))
    poly = P.cheb_coeffs(0.7, big.lambda_max_bound, 40)
    xb = torch.from_numpy(rng.normal(size=(n, d))).pin_memory()
    monkeypatch.setattr(PF, "PIPE_CHUNKS", 2)
    host = P.apply_filter(big, poly, xb.numpy())
    dev = P.apply_filter(big, poly, xb.cuda()).cpu().numpy()
    assert rel(host, dev) <= 1e-13
    monkeypatch.setattr(PF, "PIPE_MODE", "slices")
    monkeypatch.setattr(PF, "PIPE_SLICES", 8)
    assert np.array_equal(P.apply_filter(big, poly, xb.numpy()), dev)
    assert np.array_equal(P.apply_filter(big, poly, np.array(xb.numpy()[:, :37])),
                          P.apply_filter(big, poly, xb[:, :37].contiguous().cuda()).cpu().numpy())
    # a hub row past the segment cut: one final launch, then one copy
    hub = np.arange(1, 3000)
    star = P.laplacian(P.Graph(3000, np.zeros(hub.size, dtype=np.int64), hub, np.ones(hub.size)))
    xs = rng.normal(size=(3000, 16))
    ps = P.cheb_coeffs(0.7, 2.0, 12)
    assert np.array_equal(P.apply_filter(star, ps, xs), P.apply_filter(star, ps, torch.from_numpy(xs).cuda()).cpu().numpy())
