"""Device O(m) graph generators (csrc/generators.cu).

They replace the reference's O(n^2) samplers (sbm_generate graphs.py:194-221,
perturb_edges graphs.py:236-273, perturb_nodes graphs.py:276-319) for the
BASELINE sizes and are equal to them in distribution, not stream-identical.
Checked here: the exact per-block-pair edge counts the caller drew, canonical
sorted unique codes, determinism for a seed, the delete/insert list
invariants of the perturbation models, agreement of apply_delta with device
and host lists, and the model's moments (mean degree, degree dispersion,
triangle coverage, inside-block insertion share) within stated tolerances.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G(cuda_ok):
    from paper_1706_03591_b200 import generators
    return generators


def _canonical(codes, n):
    c = codes.cpu().numpy()
    assert np.all(np.diff(c) > 0), "codes must be strictly increasing"
    i, j = c // n, c % n
    assert np.all(i < j) and c.min() >= 0 and j.max() < n
    return c


def _block_of(x, n, k):
    sizes = np.full(k, n // k)
    sizes[: n % k] += 1
    return np.searchsorted(np.cumsum(sizes), x, side="right")


@pytest.mark.parametrize("n,k,s,e", [(20000, 20, 24.0, 0.05), (1003, 7, 30.0, 0.2), (50, 50, 3.0, 1.0)])
def test_planted_partition_counts_and_form(G, n, k, s, e):
    q1, q2 = G.sbm_probabilities(n, k, s, e)
    codes, m = G.planted_partition_codes_device(n, k, q1, q2, seed=11)
    c = _canonical(codes[:m], n)
    counts = G.planted_pair_counts(n, k, q1, q2, np.random.default_rng(11))
    assert m == counts.sum()
    a, b = _block_of(c // n, n, k), _block_of(c % n, n, k)
    got = np.zeros((k, k), dtype=np.int64)
    np.add.at(got, (a, b), 1)
    ia, ib = np.triu_indices(k)
    assert np.array_equal(got[ia, ib], counts)  # every pair exactly its Binomial count
    again, m2 = G.planted_partition_codes_device(n, k, q1, q2, seed=11)
    assert m2 == m and np.array_equal(again[:m].cpu().numpy(), c)  # deterministic for a seed


def test_planted_partition_moments(G):
    n, k, s = 200_000, 10, 24.0
    g, labels = G.planted_partition_device(n, k, s, 0.05, seed=3)
    c = _canonical(g.device_codes(), n)
    deg = np.bincount(c // n, minlength=n) + np.bincount(c % n, minlength=n)
    assert abs(deg.mean() - s) < 0.05 * s
    assert 0.9 < deg.var() / deg.mean() < 1.1  # Poisson-like dispersion of an SBM degree
    # inside block 0 (size 20000): pairs uniform over the strict upper triangle,
    # so 3/4 of them have their row in the first half
    size = n // k
    ii, jj = c // n, c % n
    inside = (ii < size) & (jj < size)
    frac = np.mean(ii[inside] < size // 2)
    assert abs(frac - 0.75) < 0.01
    assert abs(np.mean(jj[inside] >= size // 2) - 0.75) < 0.01


def test_planted_partition_cfg3_scale(G):
    """configs[2] size: 1M nodes, ~16M edges, generated on the device."""
    n, k = 1_000_000, 100
    q1, q2 = G.sbm_probabilities(n, k, 32.0, 0.02)
    codes, m = G.planted_partition_codes_device(n, k, q1, q2, seed=3)
    d = codes[:m]
    assert bool((d[1:] > d[:-1]).all())
    assert abs(m - 16.0e6) < 0.01 * 16.0e6


def test_chung_lu_device_matches_host_model(G):
    n, k = 200_000, 20
    args = dict(mean_degree=16.0, exponent=2.3, max_degree=2000.0, ratio=0.05)
    gd, _ = G.chung_lu_sbm_device(n, k, seed=4, **args)
    gh, _ = G.chung_lu_sbm(n, k, seed=4, **args)
    cd = _canonical(gd.device_codes(), n)
    degd = np.bincount(cd // n, minlength=n) + np.bincount(cd % n, minlength=n)
    ch = gh.edge_codes()
    degh = np.bincount(ch // n, minlength=n) + np.bincount(ch % n, minlength=n)
    assert abs(gd.m - gh.m) < 0.01 * gh.m
    assert abs(np.sort(degd)[-100:].mean() - np.sort(degh)[-100:].mean()) < 0.1 * np.sort(degh)[-100:].mean()
    assert abs(np.median(degd) - np.median(degh)) <= 1


def test_edge_churn_device_invariants(G):
    import torch
    n, k = 20000, 20
    q1, q2 = G.sbm_probabilities(n, k, 24.0, 0.05)
    g, labels = G.planted_partition_device(n, k, 24.0, 0.05, seed=1)
    codes = g.edge_codes()
    dels, ins = G.edge_churn_device(g, labels, q1, q2, 0.01, seed=7)
    dc, ic = _canonical(dels, n), _canonical(ins, n)
    count = int(round(0.01 * g.m))
    assert dc.size == ic.size and count - 5 <= dc.size <= count  # common pairs dropped from both
    assert np.all(np.isin(dc, codes)) and not np.any(np.isin(ic, codes))
    # inserts inside a block in proportion q1 * (inside pairs) : q2 * (cross pairs)
    sizes = np.bincount(labels, minlength=k)
    n_in = float((sizes * (sizes - 1) // 2).sum())
    p_in = q1 * n_in / (q1 * n_in + q2 * (n * (n - 1) / 2 - n_in))
    inside = np.mean(labels[ic // n] == labels[ic % n])
    assert abs(inside - p_in) < 5 * np.sqrt(p_in * (1 - p_in) / ic.size)
    d2, i2 = G.edge_churn_device(g, labels, q1, q2, 0.01, seed=7)
    assert torch.equal(d2, dels) and torch.equal(i2, ins)
    # apply_delta: device lists == host lists
    a = g.apply_delta(dels, ins)
    b = g.apply_delta(dc, ic)
    assert np.array_equal(a.edge_codes(), b.edge_codes())
    assert a.m == g.m - dc.size + ic.size


def test_node_switch_device_invariants(G):
    n, k = 20000, 20
    q1, q2 = G.sbm_probabilities(n, k, 24.0, 0.05)
    g, labels = G.planted_partition_device(n, k, 24.0, 0.05, seed=2)
    codes = g.edge_codes()
    dels, ins, new = G.node_switch_device(g, labels, k, q1, q2, 0.005, seed=9)
    moved = np.flatnonzero(new != labels)
    assert moved.size == int(round(0.005 * n))
    dc, ic = dels.cpu().numpy(), _canonical(ins, n)
    flag = np.zeros(n, bool)
    flag[moved] = True
    incident = codes[flag[codes // n] | flag[codes % n]]
    assert np.all(np.diff(dc) > 0) and np.all(np.isin(dc, incident))  # deletes: edges at moved nodes
    common = np.setdiff1d(incident, dc)  # redrawn edges: dropped from both lists
    assert not np.any(np.isin(ic, codes))  # inserts are absent pairs
    assert np.all(flag[ic // n] | flag[ic % n])  # every insert touches a moved node
    # expected draws: each pair with a moved endpoint once, probability by the new labels
    sizes = np.bincount(new, minlength=k)
    exp = sum(q1 * (sizes[new[u]] - 1) + q2 * (n - sizes[new[u]]) for u in moved)
    exp -= sum(q1 if new[u] == new[v] else q2 for u in moved for v in moved if v > u)  # pairs of two moved nodes once
    total = ic.size + common.size
    assert abs(total - exp) < 6 * np.sqrt(exp) + 0.02 * exp
    a = g.apply_delta(dels, ins)
    assert a.m == g.m - dc.size + ic.size
