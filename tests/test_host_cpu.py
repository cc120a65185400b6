"""CPU-only tests: C-ABI library loads and exports the header, host-side logic
mirrors the reference (validation, coefficients, RNG, tags), and the compute
path refuses to run without a GPU (no CPU fallback)."""
import numpy as np
import pytest
import torch

from conftest import golden
from oracle import csc_oracle as O


def test_library_loads_and_exports_header_symbols():
    from paper_1706_03591_b200 import _native
    lib = _native.load()
    declared = _native.header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_native.SIGNATURES) == declared
    assert lib.csc_version() >= 1


def test_status_mapping():
    from paper_1706_03591_b200 import _native
    _native.check(0, "ok")
    with pytest.raises(ValueError):
        _native.check(_native.CSC_ERR_ARG, "bad")
    with pytest.raises(_native.NativeError):
        _native.check(_native.CSC_ERR_CUDA, "cuda")


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    import paper_1706_03591_b200 as P
    with pytest.raises(RuntimeError, match="CUDA"):
        P.Graph(3, [0, 1], [1, 2], [1.0, 1.0])  # canonicalisation is device work too
    g = P.Graph(3, [], [], [])  # the empty graph needs no compute
    with pytest.raises(RuntimeError, match="CUDA"):
        P.laplacian(g)
    with pytest.raises(RuntimeError, match="CUDA"):
        P.kmeans(np.ones((4, 2)), 2)
    with pytest.raises(RuntimeError, match="CUDA"):
        P.filters._count_from_block(np.ones((4, 2)), 1.0)


def test_graph_host_validation():
    """Shape errors are raised before any device work (graphs.py:29-40)."""
    import paper_1706_03591_b200 as P
    for bad in [(4, [0, 1], [1], [1.0]), (-1, [], [], [])]:
        with pytest.raises(ValueError):
            P.Graph(*bad)


def test_oracle_canonical_order():
    """The oracle's canonicalisation (the checker of the device K9)."""
    i, j, w = O.canonical_edges(4, np.array([2, 0, 3]), np.array([0, 1, 1]), np.array([1.0, 2.0, 3.0]))
    assert i.tolist() == [0, 0, 1] and j.tolist() == [1, 2, 3] and w.tolist() == [2.0, 1.0, 3.0]


def test_coefficients_match_oracle_bitwise():
    import paper_1706_03591_b200 as P
    g = golden("small")
    assert np.array_equal(P.cheb_coeffs(1.0, 2.0, 8, damping="none").coeffs, g["c_mid_none"])
    assert np.array_equal(P.cheb_coeffs(0.3, 2.0, 12).coeffs, g["c_03_j"])
    assert np.array_equal(P.cheb_coeffs(5.0, 12.0, 12, damping="none").coeffs, g["c_5_12"])
    assert np.array_equal(P.cheb_coeffs(0.8, 2.0, 30, response="sigmoid", sigmoid_sharpness=20.0).coeffs,
                          g["c_sig"])
    assert np.array_equal(P.jackson_damping(40), g["jackson40"])
    for kw in [dict(lambda_c=0.0, lambda_max=2.0, m=10), dict(lambda_c=-0.5, lambda_max=2.0, m=10),
               dict(lambda_c=1.0, lambda_max=0.0, m=10), dict(lambda_c=1.0, lambda_max=2.0, m=0),
               dict(lambda_c=1.0, lambda_max=2.0, m=10, damping="gauss")]:
        with pytest.raises(ValueError):
            P.cheb_coeffs(**kw)
    poly = P.cheb_coeffs(2.5, 2.0, m=50, damping="none")
    assert np.allclose(poly.evaluate(np.linspace(0, 2, 100)), 1.0, atol=1e-9)


def test_random_signals_bitwise_and_validation():
    import paper_1706_03591_b200 as P
    g = golden("small")
    assert np.array_equal(P.random_signals(7, 3, seed=5), g["rs_7_3_5"])
    assert np.array_equal(P.random_signals(40, 3, seed=9, scale_dim=5), g["rs_40_3_9_sd5"])
    assert P.random_signals(7, 3, seed=5).flags["C_CONTIGUOUS"]
    with pytest.raises(ValueError):
        P.random_signals(5, 0)
    with pytest.raises(ValueError):
        P.random_signals(0, 5)


def test_feature_matrix_host_semantics():
    import paper_1706_03591_b200 as P
    fm = P.FeatureMatrix.tagged(np.zeros((4, 3)), step=2)
    assert fm.step_tags.tolist() == [2, 2, 2] and fm.stream_tags.tolist() == [0, 1, 2]
    assert fm.n == 4 and fm.d == 3
    with pytest.raises(ValueError):
        P.FeatureMatrix(np.array([[np.inf]]), np.array([0]), np.array([0]))
    with pytest.raises(ValueError):
        P.FeatureMatrix(np.zeros((4, 3)), np.array([0, 1]), np.array([0, 1]))
    assert fm.with_step(5).step_tags.tolist() == [5, 5, 5]


def test_configs_and_helpers():
    import paper_1706_03591_b200 as P
    assert P.warm_interval(0.5, 2.0) == (0.25, 1.0)
    assert P.warm_interval(1.5, 2.0) == (0.75, 2.0)
    c = P.MatvecCounter()
    c.add(3)
    c.add(4)
    assert c.count == 7
    with pytest.raises(ValueError):
        P.DynamicConfig(k=2, d=10, p=0.6)
    with pytest.raises(ValueError):
        P.DynamicConfig(k=0, d=10)
    assert P.DynamicConfig(k=2, d=207, p=0.5).reuse_count == 103
    assert P.DynamicConfig(k=2, d=10, p=0.33).reuse_count == 3
    with pytest.raises(ValueError):
        P.FilterConfig(order=0)
    with pytest.raises(ValueError):
        P.FilterConfig(precision="fp16")
    with pytest.raises(ValueError):
        P.KmeansConfig(restarts=0)


def test_laplacian_rejects_unknown_variant():
    import paper_1706_03591_b200 as P
    with pytest.raises(ValueError):
        P.laplacian(P.Graph(3, [], [], []), "random-walk")


def test_seed_states_match_numpy():
    """csc_seed_states (host restatement of SeedSequence mixing + PCG64 seeding)
    == numpy's PCG64(child).state for spawned children, incl. nested spawn keys,
    big entropy, non-default pool sizes and a partially spawned parent."""
    import numpy as np
    from numpy.random.bit_generator import _coerce_to_uint32_array
    from paper_1706_03591_b200.signals import _u32_words, child_states, column_states
    cases = [np.random.SeedSequence(0), np.random.SeedSequence(123456789),
             np.random.SeedSequence(2 ** 200 + 12345), np.random.SeedSequence([1, 2, 2 ** 40]),
             np.random.SeedSequence(7, pool_size=8), np.random.SeedSequence(5).spawn(3)[2],
             np.random.SeedSequence(9).spawn(2)[1].spawn(4)[3], np.random.SeedSequence()]
    for ss in cases:
        assert _u32_words(ss.entropy) == [int(v) for v in _coerce_to_uint32_array(ss.entropy)]
        assert _u32_words(ss.spawn_key) == [int(v) for v in _coerce_to_uint32_array(ss.spawn_key)]
        ss.spawn(5)  # partially spawned parent: children continue from n_children_spawned
        fast = child_states(ss, 37)
        ref = column_states(ss.spawn(37))
        assert np.array_equal(fast, ref)


def test_node_switch_semantics():
    """node_switch follows perturb_nodes (graphs.py:276-319): exactly round(f*n)
    nodes move to another block, every edge touching them is deleted, every
    insert touches a moved node, and moved nodes regrow their expected degree
    under the new labels."""
    import numpy as np
    from paper_1706_03591_b200 import generators as G
    n, k = 4000, 8
    q1, q2 = G.sbm_probabilities(n, k, 24.0, 0.05)
    codes = G.planted_partition_codes(n, k, q1, q2, 1)
    labels = np.repeat(np.arange(k), G.block_sizes(n, k))
    dels, ins, new = G.node_switch(codes, n, labels, k, q1, q2, 0.01, seed=5)
    moved = np.flatnonzero(new != labels)
    assert moved.size == 40 and np.all((new[moved] >= 0) & (new[moved] < k))
    mset = np.zeros(n, bool)
    mset[moved] = True
    touch = mset[codes // n] | mset[codes % n]
    # deletes are touching edges; touching edges not deleted were drawn again (cancelled)
    assert np.all(np.isin(dels, codes[touch])) and dels.size > 0.8 * touch.sum()
    assert np.all(mset[ins // n] | mset[ins % n])
    assert np.intersect1d(dels, ins).size == 0
    # expected new degree of a moved node: (block size - 1) q1 + (n - block size) q2
    nxt = np.union1d(np.setdiff1d(codes, dels, assume_unique=True), ins)
    deg = np.bincount(nxt // n, minlength=n) + np.bincount(nxt % n, minlength=n)
    sizes = np.bincount(new, minlength=k)
    expect = (sizes[new[moved]] - 1) * q1 + (n - sizes[new[moved]]) * q2
    assert abs(deg[moved].mean() - expect.mean()) < 4 * np.sqrt(expect.mean() / moved.size)
    # edge churn keeps working on the switched (non-contiguous) labels
    d2, i2 = G.edge_churn(nxt, n, new, q1, q2, 0.01, seed=6)
    same = new[i2 // n] == new[i2 % n]
    assert d2.size > 0 and 0.6 < same.mean() < 0.9  # 499 q1 : 3500 q2 -> ~0.74 same-block
