"""numpy/scipy restatement of the reference CSC hot path — TEST INFRASTRUCTURE ONLY.

Each function restates one reference function from
``/root/reference/pkg/src/cscluster`` (cited as ``file.py:line``) with plain
arrays in and out, so the tests can check the CUDA path on identical seeded
inputs without importing the reference (which does not exist on the GPU box).
The restatement is itself pinned against vectors produced by the live
reference (``tests/golden/make_golden.py`` -> ``tests/test_oracle_golden.py``).

Third-party arithmetic the reference relies on (not vendored in
``/root/reference``; ``pkg/pyproject.toml:11-12`` pins only lower bounds):
  * SciPy >= 1.10 (1.18.1 here): ``csr_matrix @ dense`` -> ``_sparsetools.csr_matvecs``
    (zero-initialised output, per-row accumulation in stored column order).
  * NumPy >= 1.24 (2.3.5 here): PCG64 + SeedSequence + ziggurat normals,
    ``Generator.choice`` (cumsum + searchsorted of one uniform), pairwise sums.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


# ---------------------------------------------------------------------------
# Chebyshev coefficients (filters.py:97-152)
# ---------------------------------------------------------------------------

def jackson(m: int) -> np.ndarray:
    """Jackson damping factors g_0..g_m (filters.py:97-104)."""
    a = np.pi / (m + 2)
    j = np.arange(m + 1)
    num = (1.0 - j / (m + 2)) * np.sin(a) * np.cos(j * a) + np.sin(j * a) * np.cos(a) / (m + 2)
    return num / np.sin(a)


def step_coeffs(lambda_c: float, lambda_max: float, m: int, damping: str = "jackson",
                response: str = "step", sharpness: float = 30.0) -> np.ndarray:
    """Coefficients c_0..c_m on x = 1 - 2 lam / lam_max (filters.py:118-152)."""
    if response == "step":
        theta = np.arccos(np.clip(1.0 - 2.0 * lambda_c / lambda_max, -1.0, 1.0))
        j = np.arange(1, m + 1)
        c = np.concatenate([[theta / np.pi], 2.0 * np.sin(j * theta) / (np.pi * j)])
    else:  # sigmoid by 4096-node Gauss-Chebyshev quadrature (filters.py:107-115, 142-146)
        num = 4096
        th = (np.arange(num) + 0.5) * np.pi / num
        lam = 0.5 * lambda_max * (1.0 - np.cos(th))
        z = np.clip(sharpness * (lam - lambda_c) / lambda_max, -60, 60)
        vals = 1.0 / (1.0 + np.exp(z))
        c = (2.0 / num) * np.cos(np.outer(np.arange(m + 1), th)) @ vals
        c[0] *= 0.5
    if damping == "jackson":
        c = c * jackson(m)
    return c


# ---------------------------------------------------------------------------
# Graph canonicalisation + Laplacian (graphs.py:29-76, 339-362)
# ---------------------------------------------------------------------------

def canonical_edges(n: int, ei, ej, ew):
    """(lo, hi, w) sorted by code lo*n+hi, stable (graphs.py:44-51)."""
    i = np.asarray(ei, dtype=np.int64).ravel()
    j = np.asarray(ej, dtype=np.int64).ravel()
    w = np.asarray(ew, dtype=np.float64).ravel()
    lo, hi = np.minimum(i, j), np.maximum(i, j)
    order = np.argsort(lo * n + hi, kind="stable")
    return lo[order], hi[order], w[order]


def degrees(n: int, lo, hi, w) -> np.ndarray:
    """bincount over the low endpoints, then plus the high endpoints (graphs.py:61-66)."""
    deg = np.bincount(lo, weights=w, minlength=n)
    deg += np.bincount(hi, weights=w, minlength=n)
    return deg


def laplacian_csr(n: int, lo, hi, w, variant: str = "normalized"):
    """Sorted CSR (indptr int32, indices int32, data f64) and the lambda_max bound.

    Restates graphs.py:339-362 without SciPy's SpGEMM: the off-diagonal value
    is ``-((inv[i] * w) * inv[j])`` (the association ``dhalf @ w @ dhalf``
    produces), the normalized diagonal is exactly 1.0 on non-isolated rows,
    the combinatorial one is the degree; explicit zeros are not stored
    (SciPy's csr - csr drops them).
    """
    lo = np.asarray(lo, dtype=np.int64)
    hi = np.asarray(hi, dtype=np.int64)
    w = np.asarray(w, dtype=np.float64)
    deg = degrees(n, lo, hi, w)
    rows = np.concatenate([lo, hi])
    cols = np.concatenate([hi, lo])
    ww = np.concatenate([w, w])
    if variant == "normalized":
        nz = deg > 0
        inv = np.where(nz, 1.0 / np.sqrt(np.where(nz, deg, 1.0)), 0.0)
        off = -((inv[rows] * ww) * inv[cols])
        diag_rows = np.flatnonzero(nz)
        diag_vals = np.ones(diag_rows.size)
        bound = 2.0
    elif variant == "combinatorial":
        off = -ww
        diag_rows = np.flatnonzero(deg != 0)
        diag_vals = deg[diag_rows]
        bound = 2.0 * float(deg.max()) if n and lo.size else 0.0
    else:
        raise ValueError(variant)
    r = np.concatenate([rows, diag_rows])
    c = np.concatenate([cols, diag_rows])
    v = np.concatenate([off, diag_vals])
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=indptr[1:])
    return indptr.astype(np.int32), c.astype(np.int32), v, bound


# ---------------------------------------------------------------------------
# Filter (filters.py:155-196)
# ---------------------------------------------------------------------------

def apply_filter(indptr, indices, data, lambda_max: float, coeffs, x) -> np.ndarray:
    """h(L) x by the three-term recurrence on M = I - (2/lambda_max) L (filters.py:155-187).

    Runs len(coeffs) - 1 SpMM blocks (never skips zero coefficients).
    """
    n = len(indptr) - 1
    a = sp.csr_matrix((np.asarray(data, np.float64), np.asarray(indices), np.asarray(indptr)),
                      shape=(n, n))
    x = np.asarray(x, dtype=np.float64)
    s = 2.0 / lambda_max
    c = np.asarray(coeffs, dtype=np.float64)
    out = c[0] * x
    t_prev, t_cur = x, x - s * (a @ x)
    out = out + c[1] * t_cur
    for cj in c[2:]:
        t_next = 2.0 * (t_cur - s * (a @ t_cur)) - t_prev
        out += cj * t_next
        t_prev, t_cur = t_cur, t_next
    return out


def count_from_block(filtered, scale: float) -> float:
    """scale * ||filtered||_F^2 (filters.py:190-196)."""
    return float((np.asarray(filtered) ** 2).sum() * scale)


def search_cutoff(filter_fn, k: int, lo: float, hi: float, lambda_max: float, order: int,
                  count_scale: float = 1.0, count_tol: float = 0.1, width_tol: float = 1e-3,
                  max_iters: int = 20, damping: str = "jackson"):
    """Bisection on the eigencount (filters.py:221-255).

    ``filter_fn(coeffs) -> filtered block`` refilters the same raw signals.
    Returns (cutoff, filtered, iterations, estimate, trace) where trace lists
    (cutoff, estimate) per probe; raises RuntimeError on non-convergence.
    """
    trace = []
    mid = est = None
    for it in range(1, max_iters + 1):
        mid = 0.5 * (lo + hi)
        filtered = filter_fn(step_coeffs(mid, lambda_max, order, damping))
        est = count_from_block(filtered, count_scale)
        trace.append((mid, est))
        if abs(est - k) <= count_tol * k:
            return mid, filtered, it, est, trace
        if est > k:
            hi = mid
        else:
            lo = mid
        if hi - lo < width_tol:
            return mid, filtered, it, est, trace
    raise RuntimeError(f"no acceptable cutoff (last {mid}, est {est})")


# ---------------------------------------------------------------------------
# Signals (signals.py:9-37)
# ---------------------------------------------------------------------------

def seed_sequence(seed) -> np.random.SeedSequence:
    return seed if isinstance(seed, np.random.SeedSequence) else np.random.SeedSequence(seed)


def random_signals(n: int, d: int, seed=0, scale_dim: int | None = None) -> np.ndarray:
    """Column c = N(0, 1/scale_dim) from SeedSequence(seed).spawn(d)[c] (signals.py:16-37)."""
    sigma = 1.0 / np.sqrt(d if scale_dim is None else int(scale_dim))
    kids = seed_sequence(seed).spawn(d)
    return np.column_stack([np.random.default_rng(ch).normal(0.0, sigma, size=n) for ch in kids])


# ---------------------------------------------------------------------------
# k-means (kmeans.py:54-144)
# ---------------------------------------------------------------------------

def sq_dists(f, c) -> np.ndarray:
    """GEMM-form squared distances clamped at 0 (kmeans.py:54-61)."""
    d2 = (f * f).sum(axis=1)[:, None] - 2.0 * f @ c.T + (c * c).sum(axis=1)[None, :]
    np.maximum(d2, 0.0, out=d2)
    return d2


_ROW_CHUNK = 1 << 14


def row_sqdist(f, c) -> np.ndarray:
    """((f - c) ** 2).sum(axis=1), the reference's expression (kmeans.py:73-76),
    evaluated in row chunks on a thread pool for large f. Each row's pairwise
    sum over its contiguous columns is the same whichever rows share the call,
    so the result is bit-identical to the one-shot expression
    (tests/test_oracle_golden.py checks it)."""
    n = f.shape[0]
    if n <= 4 * _ROW_CHUNK:
        return ((f - c) ** 2).sum(axis=1)
    from concurrent.futures import ThreadPoolExecutor
    import os
    out = np.empty(n)

    def job(a0):
        out[a0:a0 + _ROW_CHUNK] = ((f[a0:a0 + _ROW_CHUNK] - c) ** 2).sum(axis=1)

    with ThreadPoolExecutor(min(32, os.cpu_count() or 1)) as ex:
        list(ex.map(job, range(0, n, _ROW_CHUNK)))
    return out


def kmeanspp(f, k: int, rng: np.random.Generator):
    """D^2 seeding (kmeans.py:64-77). Returns (centroids, picked row indices)."""
    n = f.shape[0]
    picks = [int(rng.integers(n))]
    cent = np.empty((k, f.shape[1]))
    cent[0] = f[picks[0]]
    closest = row_sqdist(f, cent[0])
    for j in range(1, k):
        total = closest.sum()
        idx = int(rng.integers(n)) if total <= 0.0 else int(rng.choice(n, p=closest / total))
        picks.append(idx)
        cent[j] = f[idx]
        np.minimum(closest, row_sqdist(f, cent[j]), out=closest)
    return cent, picks


def lloyd(f, k: int, centroids, max_iters: int, tol: float):
    """Lloyd iterations from given centroids (kmeans.py:92-117).

    Returns (labels, cost2, history of sqrt(cost2), iterations run).
    """
    f = np.asarray(f, dtype=np.float64)
    cent = np.array(centroids, dtype=np.float64, copy=True)
    n = f.shape[0]
    prev = np.inf
    hist = []
    labels = np.zeros(n, dtype=np.int64)
    it = 0
    for it in range(1, max_iters + 1):
        d2 = sq_dists(f, cent)
        labels = d2.argmin(axis=1)
        counts = np.bincount(labels, minlength=k)
        if np.any(counts == 0):
            own = d2[np.arange(n), labels].copy()
            for j in np.flatnonzero(counts == 0):
                idx = int(own.argmax())
                labels[idx] = j
                own[idx] = -1.0
        counts = np.bincount(labels, minlength=k)
        sums = np.zeros((k, f.shape[1]))
        np.add.at(sums, labels, f)
        cent = sums / np.maximum(counts, 1)[:, None]
        cost2 = float(((f - cent[labels]) ** 2).sum())
        hist.append(np.sqrt(cost2))
        if np.isfinite(prev) and prev - cost2 <= tol * prev:
            prev = cost2
            break
        prev = cost2
    return labels, prev, hist, it


def kmeans(f, k: int, restarts: int = 10, max_iters: int = 100, tol: float = 1e-6, seed=0):
    """Best of `restarts` seeded Lloyd runs, earliest wins ties (kmeans.py:120-144).

    Returns (labels, sizes, sqrt cost).
    """
    f = np.asarray(f, dtype=np.float64)
    best = None
    for child in seed_sequence(seed).spawn(restarts):
        rng = np.random.default_rng(child)
        cent, _ = kmeanspp(f, k, rng)
        labels, cost2, _, _ = lloyd(f, k, cent, max_iters, tol)
        if best is None or cost2 < best[0]:
            best = (cost2, labels)
    cost2, labels = best
    return labels, np.bincount(labels, minlength=k), float(np.sqrt(max(cost2, 0.0)))


def adjusted_rand(a, b) -> float:
    """ARI from the contingency table (same formula as bench.py:448-460)."""
    a = np.asarray(a, dtype=np.int64)
    b = np.asarray(b, dtype=np.int64)
    ka, kb = int(a.max()) + 1, int(b.max()) + 1
    cont = np.bincount(a * kb + b, minlength=ka * kb).reshape(ka, kb).astype(np.float64)
    n = cont.sum()
    s = (cont * (cont - 1) / 2).sum()
    ra, rb = cont.sum(axis=1), cont.sum(axis=0)
    ca, cb = (ra * (ra - 1) / 2).sum(), (rb * (rb - 1) / 2).sum()
    exp = ca * cb / (n * (n - 1) / 2)
    mx = 0.5 * (ca + cb)
    if mx == exp:
        return 1.0
    return float((s - exp) / (mx - exp))


def moments(indptr, indices, data, lambda_max: float, x, m: int) -> np.ndarray:
    """mu_q = sum over columns of <x, T_q(M) x>, q = 0..2m, M = I - (2/lambda_max) L.

    Checker for the moment bisection (not a reference function; the
    reference recomputes the filtered block per probe, filters.py:237-242).
    """
    n = len(indptr) - 1
    a = sp.csr_matrix((np.asarray(data, np.float64), np.asarray(indices), np.asarray(indptr)), shape=(n, n))
    s = 2.0 / lambda_max
    x = np.asarray(x, dtype=np.float64)
    t_prev, t_cur = x, x - s * (a @ x)
    mu = [float((x * x).sum()), float((x * t_cur).sum())]
    for _ in range(2, 2 * m + 1):
        t_prev, t_cur = t_cur, 2.0 * (t_cur - s * (a @ t_cur)) - t_prev
        mu.append(float((x * t_cur).sum()))
    return np.array(mu)
