"""Pin the CPU oracle against golden vectors produced by the live reference.

The oracle (oracle/) is the checker for every GPU parity test, so it must
reproduce the reference first. Fixtures: tests/golden/make_golden.py.
"""
import numpy as np
import pytest

from conftest import golden
from oracle import csc_oracle as O
from oracle import native


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ---------------------------------------------------------------------------
# coefficients (filters.py:97-152)
# ---------------------------------------------------------------------------

def test_coefficients_bitwise():
    g = golden("small")
    assert np.array_equal(O.step_coeffs(1.0, 2.0, 8, "none"), g["c_mid_none"])
    assert np.array_equal(O.step_coeffs(0.3, 2.0, 12), g["c_03_j"])
    assert np.array_equal(O.step_coeffs(5.0, 12.0, 12, "none"), g["c_5_12"])
    assert np.array_equal(O.step_coeffs(0.8, 2.0, 30, "jackson", "sigmoid", 20.0), g["c_sig"])
    assert np.array_equal(O.jackson(40), g["jackson40"])


# ---------------------------------------------------------------------------
# Laplacian (graphs.py:29-76, 339-362): bit-exact
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["path3", "path10", "triangle", "isolated", "single", "empty",
                                  "sbm60", "weighted"])
@pytest.mark.parametrize("variant", ["normalized", "combinatorial"])
def test_laplacian_bitwise(name, variant):
    g = golden("small")
    n = int(g[f"{name}_n"])
    lo, hi, w = O.canonical_edges(n, g[f"{name}_i"], g[f"{name}_j"], g[f"{name}_w"])
    indptr, indices, data, bound = O.laplacian_csr(n, lo, hi, w, variant)
    p = f"{name}_{variant}"
    assert np.array_equal(indptr, g[f"{p}_indptr"])
    assert np.array_equal(indices, g[f"{p}_indices"])
    assert np.array_equal(data, g[f"{p}_data"])
    assert bound == float(g[f"{p}_bound"])


def test_laplacian_cfg1_bitwise():
    g = golden("cfg1")
    lo, hi, w = O.canonical_edges(1000, g["g_i"], g["g_j"], g["g_w"])
    indptr, indices, data, bound = O.laplacian_csr(1000, lo, hi, w)
    assert np.array_equal(indptr, g["L_indptr"])
    assert np.array_equal(indices, g["L_indices"])
    assert np.array_equal(data, g["L_data"])
    assert indices.size == 20844


# ---------------------------------------------------------------------------
# signals (signals.py:16-37): bitwise
# ---------------------------------------------------------------------------

def test_random_signals_bitwise():
    g = golden("small")
    assert np.array_equal(O.random_signals(7, 3, 5), g["rs_7_3_5"])
    assert np.array_equal(O.random_signals(40, 3, 9, scale_dim=5), g["rs_40_3_9_sd5"])
    c = golden("cfg1")
    sig = np.random.SeedSequence(0).spawn(2)[0]
    assert np.array_equal(O.random_signals(1000, 40, sig), c["R"])


# ---------------------------------------------------------------------------
# filter (filters.py:155-196)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("tag", ["m37", "m40none", "sig60", "ident", "lin", "allpass"])
def test_filter_numpy_oracle_bitwise(tag):
    g = golden("small")
    out = O.apply_filter(g["sbm60_normalized_indptr"], g["sbm60_normalized_indices"],
                         g["sbm60_normalized_data"], float(g[f"f60_{tag}_lmax"]),
                         g[f"f60_{tag}_coeffs"], g["f60_x"])
    assert np.array_equal(out, g[f"f60_{tag}_out"])


@pytest.mark.parametrize("tag", ["m37", "m40none", "sig60", "ident", "lin", "allpass"])
def test_filter_c_oracle_matches(tag):
    g = golden("small")
    out = native.cheb_filter(g["sbm60_normalized_indptr"], g["sbm60_normalized_indices"],
                             g["sbm60_normalized_data"], float(g[f"f60_{tag}_lmax"]),
                             g[f"f60_{tag}_coeffs"], g["f60_x"])
    assert np.array_equal(out, g[f"f60_{tag}_out"])   # bitwise: same op order, no FMA


def test_filter_cfg1_c_oracle_and_threads():
    g = golden("cfg1")
    args = (g["L_indptr"], g["L_indices"], g["L_data"], 2.0, g["coeffs_05"], g["R"])
    one = native.cheb_filter(*args, nthreads=1)
    many = native.cheb_filter(*args, nthreads=4)
    assert np.array_equal(one, many)           # row split never changes a bit
    assert np.array_equal(one, g["filt_05"])
    assert np.array_equal(O.apply_filter(g["L_indptr"], g["L_indices"], g["L_data"], 2.0,
                                         g["coeffs_05"], g["R"]), g["filt_05"])


def test_filter_combinatorial_weighted():
    g = golden("small")
    out = O.apply_filter(g["weighted_combinatorial_indptr"], g["weighted_combinatorial_indices"],
                         g["weighted_combinatorial_data"], float(g["fw_lmax"]), g["fw_coeffs"], g["fw_x"])
    assert np.array_equal(out, g["fw_out"])


def test_bisection_trace_cfg1():
    g = golden("cfg1")
    ip, ix, dv = g["L_indptr"], g["L_indices"], g["L_data"]
    r = g["R"]
    cut, filt, iters, est, trace = O.search_cutoff(
        lambda c: O.apply_filter(ip, ix, dv, 2.0, c, r), 10, 0.0, 2.0, 2.0, 50, max_iters=8)
    assert [t[0] for t in trace] == list(g["probe_cutoffs"])
    np.testing.assert_allclose([t[1] for t in trace], g["probe_estimates"], rtol=1e-12)
    assert cut == float(g["cutoff"]) and iters == int(g["iters"])
    assert np.array_equal(filt, g["features"])


def test_find_lambda_k_trace_small():
    g = golden("small")
    ip, ix, dv = (g[f"sbm60_normalized_{k}"] for k in ("indptr", "indices", "data"))
    r = O.random_signals(60, 12, 5)
    cut, filt, iters, est, trace = O.search_cutoff(
        lambda c: O.apply_filter(ip, ix, dv, 2.0, c, r), 3, 0.0, 2.0, 2.0, 40)
    assert [t[0] for t in trace] == list(g["flk_cutoffs"])
    assert cut == float(g["flk_lambda"]) and iters == int(g["flk_iters"])
    assert np.array_equal(filt, g["flk_features"])


# ---------------------------------------------------------------------------
# k-means (kmeans.py:54-144)
# ---------------------------------------------------------------------------

def test_kmeanspp_and_lloyd_cfg1():
    g = golden("cfg1")
    f = g["features"]
    child = np.random.SeedSequence(0).spawn(2)[1].spawn(1)[0]
    cent, picks = O.kmeanspp(f, 10, np.random.default_rng(child))
    assert np.array_equal(cent, g["km_init"])
    labels, cost2, hist, _ = O.lloyd(f, 10, cent, 20, 1e-6)
    assert np.array_equal(labels, g["km_labels"])
    assert cost2 == float(g["km_cost2"])
    assert np.array_equal(hist, g["km_hist"])


def test_kmeans_restarts_golden():
    g = golden("kmeans")
    labels, sizes, cost = O.kmeans(g["a_f"], 3, seed=123)
    assert np.array_equal(labels, g["a_labels"]) and cost == float(g["a_cost"])
    for s in range(6):
        labels, _, cost = O.kmeans(np.array([[0.0], [0.0], [5.0]]), 3, restarts=1, seed=s)
        assert np.array_equal(labels, g[f"dup{s}_labels"]) and cost == float(g[f"dup{s}_cost"])
    labels, _, cost = O.kmeans(g["b_f"], 12, restarts=3, max_iters=50, seed=77)
    assert np.array_equal(labels, g["b_labels"]) and cost == float(g["b_cost"])


def test_adjusted_rand_identity():
    a = np.array([0, 0, 1, 1, 2, 2])
    assert O.adjusted_rand(a, a) == 1.0
    assert O.adjusted_rand(a, np.array([1, 1, 0, 0, 2, 2])) == 1.0


def test_row_sqdist_chunked_is_bitwise():
    """The oracle's threaded row-chunked D^2 equals the reference's one-shot expression."""
    rng = np.random.default_rng(5)
    f = rng.standard_normal((300_000, 37))
    c = f[11]
    assert np.array_equal(O.row_sqdist(f, c), ((f - c) ** 2).sum(axis=1))


def test_high_order_filters_bitwise():
    """m = 300 / m = 250 cases of the reference's own tests (test_filters.py:178-184, 277-291)."""
    g = golden("high_order")
    ip, ix, dv = g["l300_indptr"], g["l300_indices"], g["l300_data"]
    n = len(ip) - 1
    assert np.array_equal(O.step_coeffs(float(g["g300_cut"]), 2.0, 300), g["g300_coeffs"])
    r = O.random_signals(n, 100, 0)
    out = native.cheb_filter(ip, ix, dv, 2.0, g["g300_coeffs"], r)
    assert np.array_equal(out, g["g300_feats0"])
    assert O.count_from_block(out, 1.0) == float(g["g300_ests"][0])
    ip, ix, dv = g["l120_indptr"], g["l120_indices"], g["l120_data"]
    for tag in ("mid", "eig"):
        c = O.step_coeffs(float(g[f"g120_{tag}_cut"]), 2.0, 250)
        assert np.array_equal(O.apply_filter(ip, ix, dv, 2.0, c, g["g120_r"]), g[f"g120_{tag}_approx"])
