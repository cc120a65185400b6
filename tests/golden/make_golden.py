"""Generate golden vectors by running the LIVE reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--skip-cfg2]

Imports ``cscluster`` from ``/root/reference/pkg/src`` (read-only), runs its
public functions on seeded inputs and writes compressed ``.npz`` fixtures next
to this script. The fixtures travel with the repo; ``/root/reference`` does
not exist on the GPU box and nothing else reads it.

To record the per-probe bisection trace, the reference's module-level
``cheb_coeffs`` / ``_count_from_block`` names are wrapped (observers only: the
wrapped functions are called unchanged and their results passed through).
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)

import cscluster as cc  # noqa: E402
from cscluster import dynamic as ref_dynamic  # noqa: E402
from cscluster import filters as ref_filters  # noqa: E402
from cscluster.kmeans import _kmeanspp_init, _lloyd  # noqa: E402


class ProbeRecorder:
    """Observe cheb_coeffs cutoffs and _count_from_block estimates."""

    def __init__(self):
        self.cutoffs, self.estimates = [], []
        self._orig_cc = ref_filters.cheb_coeffs
        self._orig_cnt = ref_filters._count_from_block
        self._orig_dyn_cnt = ref_dynamic._count_from_block

    def __enter__(self):
        rec = self

        def cheb(*a, **kw):
            rec.cutoffs.append(float(a[0]) if a else float(kw["lambda_c"]))
            return rec._orig_cc(*a, **kw)

        def cnt(filtered, scale):
            v = rec._orig_cnt(filtered, scale)
            rec.estimates.append(v)
            return v

        ref_filters.cheb_coeffs = cheb
        ref_filters._count_from_block = cnt
        ref_dynamic._count_from_block = cnt
        return self

    def __exit__(self, *exc):
        ref_filters.cheb_coeffs = self._orig_cc
        ref_filters._count_from_block = self._orig_cnt
        ref_dynamic._count_from_block = self._orig_dyn_cnt


def lap_arrays(prefix, lap):
    m = lap.matrix
    return {f"{prefix}_indptr": m.indptr.astype(np.int32), f"{prefix}_indices": m.indices.astype(np.int32),
            f"{prefix}_data": m.data.astype(np.float64), f"{prefix}_bound": np.float64(lap.lambda_max_bound)}


def graph_arrays(prefix, g):
    return {f"{prefix}_n": np.int64(g.n), f"{prefix}_i": g.edge_i.astype(np.int32),
            f"{prefix}_j": g.edge_j.astype(np.int32), f"{prefix}_w": g.edge_w.astype(np.float64)}


# ---------------------------------------------------------------------------

def make_cfg1():
    """BASELINE.json configs[0]: static CSC, SBM n=1000, k=10, d=40, m=50, 8 probes max."""
    params = cc.SbmParams(n=1000, k=10, s=19.62, e=1 / 90)
    g, planted = cc.sbm_generate(params, 0)
    lap = cc.laplacian(g)
    out = {**graph_arrays("g", g), **lap_arrays("L", lap), "planted": planted.astype(np.int32),
           "q1": np.float64(params.q1), "q2": np.float64(params.q2)}

    ss = np.random.SeedSequence(0)
    sig_ss, km_ss = ss.spawn(2)
    r = cc.random_signals(1000, 40, sig_ss)
    out["R"] = r
    fcfg = cc.FilterConfig(order=50, max_iters=8)
    with ProbeRecorder() as rec:
        cutoff, filtered, poly, iters, est = ref_filters._search_cutoff(
            lap, 10, r, (0.0, 2.0), fcfg, None, 1.0)
    out.update(probe_cutoffs=np.array(rec.cutoffs), probe_estimates=np.array(rec.estimates),
               cutoff=np.float64(cutoff), iters=np.int64(iters), est=np.float64(est),
               coeffs=poly.coeffs, features=filtered)
    # fixed-cutoff filter (cutoff 0.5, m=50) of the raw block
    p05 = cc.cheb_coeffs(0.5, 2.0, 50)
    out["coeffs_05"] = p05.coeffs
    out["filt_05"] = cc.apply_filter(lap, p05, r)

    # k-means: restarts=1, max_iters=20 (configs[0]); init centroids from the stream
    km_child = np.random.SeedSequence(0).spawn(2)[1].spawn(1)[0]
    init = _kmeanspp_init(filtered, 10, np.random.default_rng(km_child))
    labels, cost2, hist = _lloyd(filtered, 10, np.random.default_rng(km_child), 20, 1e-6)
    out.update(km_init=init, km_labels=labels.astype(np.int32), km_cost2=np.float64(cost2),
               km_hist=np.array(hist))

    counter = cc.MatvecCounter()
    a, diag = cc.csc_assign(lap, 10, 40, filter_cfg=fcfg,
                            kmeans_cfg=cc.KmeansConfig(restarts=1, max_iters=20), seed=0,
                            counter=counter)
    out.update(csc_labels=a.labels.astype(np.int32), csc_cost=np.float64(a.feature_cost),
               csc_lambda=np.float64(diag.lambda_k), csc_iters=np.int64(diag.search_iters),
               csc_matvecs=np.int64(diag.matvecs))
    # default (10-restart) k-means on the accepted features
    a10 = cc.kmeans(filtered, 10, cc.KmeansConfig(), seed=5)
    out.update(km10_labels=a10.labels.astype(np.int32), km10_cost=np.float64(a10.feature_cost))
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **out)


def _sbm60(seed):
    params = cc.SbmParams(n=60, k=3, s=10, e=0.2)
    g, _ = cc.sbm_generate(params, seed)
    return g


def make_small():
    out = {}
    P = lambda n: cc.Graph(n, np.arange(n - 1), np.arange(1, n), np.ones(n - 1))  # noqa: E731
    graphs = {
        "path3": P(3),
        "path10": P(10),
        "triangle": cc.Graph(3, [0, 1, 0], [1, 2, 2], [1.0, 1.0, 1.0]),
        "isolated": cc.Graph(4, [0, 1], [1, 2], [1.0, 1.0]),
        "single": cc.Graph(5, [0], [1], [1.0]),
        "empty": cc.Graph(10, [], [], []),
        "sbm60": _sbm60(0),
    }
    rng = np.random.default_rng(42)
    # weighted graph with isolated nodes and unsorted / reversed input pairs
    n = 80
    iu, ju = np.triu_indices(n - 5, 1)
    pick = rng.random(iu.size) < 0.08
    ii, jj = iu[pick], ju[pick]
    flip = rng.random(ii.size) < 0.5
    ii, jj = np.where(flip, jj, ii), np.where(flip, ii, jj)
    perm = rng.permutation(ii.size)
    graphs["weighted"] = cc.Graph(n, ii[perm], jj[perm], rng.uniform(0.1, 3.0, ii.size))
    for name, g in graphs.items():
        out.update(graph_arrays(name, g))
        for variant in ("normalized", "combinatorial"):
            out.update(lap_arrays(f"{name}_{variant}", cc.laplacian(g, variant)))

    lap = cc.laplacian(graphs["sbm60"])
    x = np.random.default_rng(4).normal(size=(60, 6))
    out["f60_x"] = x
    for tag, poly in {
        "m37": cc.cheb_coeffs(0.5, lap.lambda_max_bound, m=37),
        "m40none": cc.cheb_coeffs(0.7, lap.lambda_max_bound, m=40, damping="none"),
        "sig60": cc.cheb_coeffs(1.0, 2.0, m=60, damping="none", response="sigmoid"),
        "ident": cc.FilterPoly(5, np.array([1.0, 0, 0, 0, 0, 0]), 1.0, 2.0, "none"),
        "lin": cc.FilterPoly(1, np.array([1.0, -1.0]), 1.0, 2.0, "none"),
        "allpass": cc.cheb_coeffs(2.5, 2.0, m=50, damping="none"),
    }.items():
        out[f"f60_{tag}_coeffs"] = poly.coeffs
        out[f"f60_{tag}_lmax"] = np.float64(poly.lambda_max)
        out[f"f60_{tag}_out"] = cc.apply_filter(lap, poly, x)
    # weighted-graph filter, combinatorial variant (lambda_max = 2 max deg)
    lapc = cc.laplacian(graphs["weighted"], "combinatorial")
    xw = np.random.default_rng(5).normal(size=(n, 3))
    pw = cc.cheb_coeffs(0.3 * lapc.lambda_max_bound, lapc.lambda_max_bound, m=30)
    out.update(fw_x=xw, fw_coeffs=pw.coeffs, fw_lmax=np.float64(pw.lambda_max),
               fw_out=cc.apply_filter(lapc, pw, xw))

    # coefficient known answers
    for tag, kw in {
        "c_mid_none": dict(lambda_c=1.0, lambda_max=2.0, m=8, damping="none"),
        "c_03_j": dict(lambda_c=0.3, lambda_max=2.0, m=12),
        "c_5_12": dict(lambda_c=5.0, lambda_max=12.0, m=12, damping="none"),
        "c_sig": dict(lambda_c=0.8, lambda_max=2.0, m=30, response="sigmoid", sigmoid_sharpness=20.0),
    }.items():
        out[tag] = cc.cheb_coeffs(**kw).coeffs
    out["jackson40"] = cc.jackson_damping(40)

    # find_lambda_k on the 60-node SBM: trace + features
    with ProbeRecorder() as rec:
        lam, feats, iters = cc.find_lambda_k(lap, 3, d=12, m=40, seed=5)
    out.update(flk_cutoffs=np.array(rec.cutoffs), flk_estimates=np.array(rec.estimates),
               flk_lambda=np.float64(lam), flk_iters=np.int64(iters), flk_features=feats.values)

    # random signals
    out["rs_7_3_5"] = cc.random_signals(7, 3, seed=5)
    out["rs_40_3_9_sd5"] = cc.random_signals(40, 3, seed=9, scale_dim=5)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)


def make_kmeans():
    out = {}
    rng = np.random.default_rng(2)
    f = rng.normal(size=(50, 4))
    a = cc.kmeans(f, 3, seed=123)
    out.update(a_f=f, a_labels=a.labels.astype(np.int32), a_cost=np.float64(a.feature_cost))
    dup = np.array([[0.0], [0.0], [5.0]])
    for s in range(6):
        b = cc.kmeans(dup, 3, cc.KmeansConfig(restarts=1), seed=s)
        out[f"dup{s}_labels"] = b.labels.astype(np.int32)
        out[f"dup{s}_cost"] = np.float64(b.feature_cost)
    rect = np.array([[0.0, 0.0], [2.0, 0.0], [0.0, 0.1], [2.0, 0.1]])
    r = cc.kmeans(rect, 2, cc.KmeansConfig(restarts=10), seed=0)
    out.update(rect_labels=r.labels.astype(np.int32), rect_cost=np.float64(r.feature_cost))
    # blobs big enough to exercise the GPU tiles (n=3000, d=24, k=12)
    centers = rng.normal(scale=4.0, size=(12, 24))
    lab = rng.integers(0, 12, size=3000)
    fb = centers[lab] + rng.normal(size=(3000, 24))
    kb = cc.kmeans(fb, 12, cc.KmeansConfig(restarts=3, max_iters=50), seed=77)
    child = np.random.SeedSequence(77).spawn(3)[0]
    init = _kmeanspp_init(fb, 12, np.random.default_rng(child))
    lb, c2, hist = _lloyd(fb, 12, np.random.default_rng(child), 50, 1e-6)
    out.update(b_f=fb, b_labels=kb.labels.astype(np.int32), b_cost=np.float64(kb.feature_cost),
               b_init=init, b_r0_labels=lb.astype(np.int32), b_r0_cost2=np.float64(c2),
               b_r0_hist=np.array(hist))
    np.savez_compressed(os.path.join(HERE, "kmeans.npz"), **out)


def make_dynamic_small():
    params = cc.SbmParams(n=300, k=4, s=25, e=1 / 6)
    graphs, labels = cc.perturbed_sequence(params, 4, 0.03, 0.01, seed=9)
    cfg = cc.DynamicConfig(k=4, d=40, p=0.5, filter=cc.FilterConfig(order=60),
                           kmeans=cc.KmeansConfig(restarts=6))
    out = {}
    for t, g in enumerate(graphs):
        out.update(graph_arrays(f"g{t}", g))
    a, state, diag = cc.dynamic_init(graphs[0], cfg, seed=10)
    steps = [(a, state, diag)]
    for g in graphs[1:]:
        a, state, diag = cc.dynamic_step(state, g, cfg)
        steps.append((a, state, diag))
    for t, (a, st, dg) in enumerate(steps):
        out.update({f"s{t}_labels": a.labels.astype(np.int32), f"s{t}_cost": np.float64(a.feature_cost),
                    f"s{t}_lambda": np.float64(dg.lambda_k), f"s{t}_refined": np.bool_(dg.refined),
                    f"s{t}_iters": np.int64(dg.search_iters), f"s{t}_reused": np.int64(dg.reused),
                    f"s{t}_mv_fresh": np.int64(dg.matvecs_fresh), f"s{t}_mv_total": np.int64(dg.matvecs_total),
                    f"s{t}_features": st.features.values, f"s{t}_step_tags": st.features.step_tags,
                    f"s{t}_stream_tags": st.features.stream_tags})
    np.savez_compressed(os.path.join(HERE, "dynamic_small.npz"), **out)


def make_cfg2(steps=2):
    """BASELINE.json configs[1] (n=20k, k=20, d=80, p=0.5, m=60): init + first steps.

    Stores graph 1, the per-step insert/delete code lists, and per-step
    summaries (estimates, cutoff, labels, cost, column norms, a row sample).
    """
    params = cc.SbmParams(n=20000, k=20, s=24, e=0.05)
    t0 = time.time()
    graphs, _ = cc.perturbed_sequence(params, steps + 1, 0.01, 0.005, seed=0)
    print(f"cfg2 sequence: {time.time() - t0:.1f}s", flush=True)
    cfg = cc.DynamicConfig(k=20, d=80, p=0.5, filter=cc.FilterConfig(order=60))
    out = {**graph_arrays("g0", graphs[0])}
    for t in range(1, len(graphs)):
        prev, cur = graphs[t - 1].edge_codes(), graphs[t].edge_codes()
        out[f"del{t}"] = np.setdiff1d(prev, cur, assume_unique=True)
        out[f"ins{t}"] = np.setdiff1d(cur, prev, assume_unique=True)
    rows = np.arange(0, 20000, 313)
    with ProbeRecorder() as rec:
        a, state, diag = cc.dynamic_init(graphs[0], cfg, seed=0)
        n0 = len(rec.estimates)
        res = [(a, state, diag, list(rec.cutoffs), list(rec.estimates))]
        for g in graphs[1:]:
            c0, e0 = len(rec.cutoffs), len(rec.estimates)
            a, state, diag = cc.dynamic_step(state, g, cfg)
            res.append((a, state, diag, rec.cutoffs[c0:], rec.estimates[e0:]))
    assert n0 > 0
    out["rows"] = rows
    for t, (a, st, dg, cuts, ests) in enumerate(res):
        v = st.features.values
        out.update({f"s{t}_labels": a.labels.astype(np.int16), f"s{t}_cost": np.float64(a.feature_cost),
                    f"s{t}_lambda": np.float64(dg.lambda_k), f"s{t}_refined": np.bool_(dg.refined),
                    f"s{t}_iters": np.int64(dg.search_iters), f"s{t}_mv_total": np.int64(dg.matvecs_total),
                    f"s{t}_cutoffs": np.array(cuts), f"s{t}_estimates": np.array(ests),
                    f"s{t}_colnorm2": (v ** 2).sum(axis=0), f"s{t}_rowsample": v[rows],
                    f"s{t}_stream_tags": st.features.stream_tags, f"s{t}_step_tags": st.features.step_tags,
                    f"s{t}_wall_ms": np.float64(dg.wall_ms)})
    np.savez_compressed(os.path.join(HERE, "cfg2.npz"), **out)
    print(f"cfg2 total: {time.time() - t0:.1f}s", flush=True)


def make_high_order():
    """High-order filters of the reference's own tests: m = 300 eigencounts on the
    sbm300 fixture (pkg/tests/test_filters.py:178-184, conftest.py:33-38) and the
    m = 250 approximation of the ideal projector (test_filters.py:277-291)."""
    out = {}
    params = cc.SbmParams(n=300, k=4, s=25, e=1 / 6)
    g, _ = cc.sbm_generate(params, seed=2024)
    lap = cc.laplacian(g)
    out.update(graph_arrays("g300", g))
    out.update(lap_arrays("l300", lap))
    basis = cc.eigendecompose(lap, 4)
    cut = 0.5 * (basis.eigenvalues[-1] + basis.lambda_next)
    out["g300_cut"] = np.float64(cut)
    ests, feats = [], []
    for s in range(5):
        est, fm = cc.eigencount(lap, cut, d=100, m=300, seed=s)
        ests.append(est)
        if s == 0:
            feats = fm.values
    out["g300_ests"] = np.array(ests)
    out["g300_feats0"] = feats
    poly = cc.cheb_coeffs(cut, lap.lambda_max_bound, 300)
    out["g300_coeffs"] = poly.coeffs
    params = cc.SbmParams(n=120, k=3, s=12, e=0.1)
    g, _ = cc.sbm_generate(params, 11)
    lap = cc.laplacian(g)
    out.update(graph_arrays("g120", g))
    out.update(lap_arrays("l120", lap))
    basis = cc.eigendecompose(lap, 3)
    r = cc.random_signals(120, 40, seed=12)
    grid = np.linspace(0.0, lap.lambda_max_bound, 4000)
    for tag, cut in (("mid", 0.5 * (basis.eigenvalues[-1] + basis.lambda_next)), ("eig", basis.eigenvalues[-1])):
        poly = cc.cheb_coeffs(cut, lap.lambda_max_bound, m=250, damping="jackson")
        out[f"g120_{tag}_cut"] = np.float64(cut)
        out[f"g120_{tag}_approx"] = cc.apply_filter(lap, poly, r)
        out[f"g120_{tag}_ideal"] = cc.ideal_projector_apply(basis, r)
        step = (grid <= cut).astype(np.float64)
        out[f"g120_{tag}_worst"] = np.float64(np.abs(poly.evaluate(grid) - step).max())
    out["g120_r"] = r
    np.savez_compressed(os.path.join(HERE, "high_order.npz"), **out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-cfg2", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    jobs = {"cfg1": make_cfg1, "small": make_small, "kmeans": make_kmeans,
            "dynamic_small": make_dynamic_small, "cfg2": make_cfg2, "high_order": make_high_order}
    for name, fn in jobs.items():
        if args.only and name not in args.only.split(","):
            continue
        if name == "cfg2" and args.skip_cfg2:
            continue
        t = time.time()
        fn()
        print(f"{name}: {time.time() - t:.1f}s", flush=True)
