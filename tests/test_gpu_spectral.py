"""Spectral known answers of the filter and the eigencount (filters.py:155-213)
on the GPU path, checked against a dense eigendecomposition of the Laplacian
(numpy eigh: test infrastructure only, small graphs).

- h(L) x from apply_filter equals U diag(p(lambda)) U^T x, p the filter's
  Chebyshev polynomial on the eigenvalues (relative 1e-8).
- eigencount at the spectrum's top (lambda_c = lambda_max) keeps every
  component: its estimate is ||R||_F^2 (to rounding).
- eigencount is non-decreasing in lambda_c for Jackson damping (the damped
  step is a positive-kernel smoothing of a monotone step).
- the count at a cutoff equals sum_i p(lambda_i)^2 ||U^T R e_i||^2 (the
  dense form of the same estimator).
"""
import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(cuda_ok):
    import paper_1706_03591_b200 as P
    return P


def small_graph(P, name="sbm60"):
    g = golden("small")
    return P.Graph(int(g[f"{name}_n"]), g[f"{name}_i"], g[f"{name}_j"], g[f"{name}_w"])


@pytest.mark.parametrize("variant,cut,m", [("normalized", 0.4, 30), ("normalized", 1.1, 60),
                                           ("combinatorial", 3.0, 40)])
def test_filter_equals_dense_spectral_form(P, variant, cut, m):
    lap = P.laplacian(small_graph(P, "sbm60" if variant == "normalized" else "weighted"), variant)
    L = lap.matrix.toarray()
    lam, U = np.linalg.eigh(L)
    poly = P.cheb_coeffs(min(cut, lap.lambda_max_bound), lap.lambda_max_bound, m)
    x = np.random.default_rng(m).normal(size=(lap.n, 5))
    got = P.apply_filter(lap, poly, x)
    ref = U @ (poly.evaluate(lam)[:, None] * (U.T @ x))
    assert np.linalg.norm(got - ref) <= 1e-8 * np.linalg.norm(ref)


def test_eigencount_top_keeps_everything(P):
    lap = P.laplacian(small_graph(P))
    est, feats = P.eigencount(lap, lap.lambda_max_bound, 16, m=40, seed=3)
    raw = P.random_signals(lap.n, 16, 3)
    assert np.allclose(feats.values, raw, rtol=0, atol=1e-12)
    assert abs(est - float((raw ** 2).sum())) <= 1e-12 * est


def test_eigencount_monotone_and_dense_form(P):
    lap = P.laplacian(small_graph(P))
    lam, U = np.linalg.eigh(lap.matrix.toarray())
    d = 24
    R = P.random_signals(lap.n, d, 5)
    energy = ((U.T @ R) ** 2).sum(axis=1)  # per eigenvector
    cuts = np.linspace(0.05, 1.95, 12)
    ests = []
    for c in cuts:
        est, _ = P.eigencount(lap, float(c), d, m=50, seed=5)
        poly = P.cheb_coeffs(float(c), lap.lambda_max_bound, 50)
        dense = float((poly.evaluate(lam) ** 2 * energy).sum())
        assert abs(est - dense) <= 1e-9 * max(dense, 1e-300) + 1e-12
        ests.append(est)
    assert all(b >= a - 1e-9 * max(abs(a), 1.0) for a, b in zip(ests, ests[1:]))
