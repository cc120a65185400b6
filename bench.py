#!/usr/bin/env python
"""Benchmark of the CSC Chebyshev-filter hot path on B200 (one JSON line on stdout).

Headline (BASELINE.json metric): filtered nnz*d*order per second, with the
fused SpMM sweep's fraction of the HBM roofline, and ms per dynamic-CSC step.

Workload (N=1, `--workload cfg3`, the SpMM roofline config of BASELINE.json
configs[2]): planted partition n=1,000,000, k=100 blocks, mean degree 32,
p_out/p_in=0.02 (nnz(L) ~ 33.0M, int32 CSR), d=128 N(0,1/d) signals, fp64,
Chebyshev order m=100. One step = one apply_filter (100 fused SpMM sweeps) of
the device-resident block. Inputs (1 GB signals + 2 GB recurrence buffers)
exceed the 126 MB L2, so no explicit flush is needed between steps.

Also on the same line (each untimed by the headline's clock):
  * e2e: the public apply_filter with host numpy in / numpy out, pinned
    (the contract's headline e2e) and pageable (an ordinary numpy array), >= 5
    calls each;
  * variants.fp32 (cfg3) and variants.cfg4_fp32 / cfg4_fp64 (BASELINE
    configs[3]: Chung-Lu n = 4M, skewed degrees, d = 64, m = 80): throughput,
    sweep roofline on the minimum bytes, fp32 error vs fp64;
  * dynamic (configs[1]) and dynamic_cfg5 (configs[4], p = 0.5, 1% churn, plus
    `matrix`: churn {0.1, 1, 5}% x p {0, 0.25, 0.5} sampled, quality vs p = 0):
    ms per step with the host insert/delete lists merged on the device inside
    the timed step, phase split, and one refined step;
  * cpu_baseline: the C restatement on all host cores (the `--impl reference`
    arm) and the unmodified reference's own apply_filter (SciPy, installed in
    baseline/_ref) on the same sample.

Multi-GPU (torchrun): the filter shards by columns with no exchange
(filters.py:159-161); every rank filters its own d=128 block of the same
graph ("scaling": "weak"), time = max over ranks.

`--impl reference`: the reference's CPU path for the same workload — the
C restatement of apply_filter (oracle/cheb_filter.c, bit-identical to the
reference on the golden vectors) on all host cores, a bounded sample of 2
orders per step, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "cfg3": dict(n=1_000_000, k=100, deg=32.0, ratio=0.02, d=128, order=100, cutoff=0.05, seed=3),
    "cfg1": dict(n=1000, k=10, deg=19.62, ratio=1 / 90, d=40, order=50, cutoff=0.5, seed=0),
    "cfg5": dict(n=2_000_000, k=64, deg=20.0, ratio=0.05, d=96, order=80, cutoff=0.05, seed=5),
}
CFG4 = dict(n=4_000_000, k=50, deg=16.0, exponent=2.3, max_degree=20000.0, ratio=0.05, d=64, order=80,
            cutoff=0.05, seed=4)
METRIC = "filtered nnz*d*order/s"
UNIT = "nnz*d*order/s"


def traffic_capture(workload: str, precision: str):
    """The committed ncu capture of this workload's sweep: DRAM bytes per launch
    plus the kernel instance, grid and commit it was taken of
    (profiles/r02_sweep_<workload>_<precision>.json, written by
    tools/capture_traffic.py), or None."""
    path = os.path.join(ROOT, "profiles", f"r02_sweep_{workload}_{precision}.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        cap = json.load(fh)
    cap["source"] = os.path.relpath(path, ROOT)
    return cap


def last_launch(lib):
    buf = ctypes.create_string_buffer(128)
    grid = ctypes.c_int(0)
    lib.csc_sweep_last_launch(buf, 128, ctypes.byref(grid))
    return buf.value.decode(), int(grid.value)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def make_graph_codes(w):
    from paper_1706_03591_b200 import generators as G
    q1, q2 = G.sbm_probabilities(w["n"], w["k"], w["deg"], w["ratio"])
    return G.planted_partition_codes(w["n"], w["k"], q1, q2, w["seed"]), (q1, q2)


def b_min(n, nnz, d, s):
    """SURVEY 8(d) minimum bytes of one sweep: CSR (indptr, indices, values),
    one gathered d-row per stored entry, the written T_{j+1} rows."""
    return 4 * (n + 1) + nnz * (4 + s) + nnz * d * s + n * d * s


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx = [], []
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_filter_sample(indptr, indices, data, r, coeffs, orders=2, threads=0):
    """Time `orders` SpMM blocks of the C restatement (the reference's CPU path)."""
    from oracle import native as ON
    c = np.ascontiguousarray(coeffs[: orders + 1])
    t0 = time.perf_counter()
    ON.cheb_filter(indptr, indices, data, 2.0, c, r, nthreads=threads)
    return time.perf_counter() - t0, (threads or ON.num_threads())


def reference_scipy_sample(matrix, r, coeffs, orders=2):
    """Time `orders` SpMM blocks of the UNMODIFIED reference's apply_filter
    (cscluster from baseline/_ref: SciPy csr_matvecs, single-threaded), or None
    when the reference is not installed."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "cscluster")):
        return None
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    try:
        import cscluster as cc
        from cscluster.graphs import LaplacianMatrix as RefLap
    except Exception:
        return None
    lap = RefLap(matrix, "normalized", 2.0)
    c = np.ascontiguousarray(coeffs[: orders + 1])
    poly = cc.FilterPoly(orders, c, 0.05, 2.0, "jackson")
    t0 = time.perf_counter()
    cc.apply_filter(lap, poly, r)
    return time.perf_counter() - t0


def workload_desc(name, w, n, d, order):
    """config.workload of both arms (the same string)."""
    return (f"{name}: planted partition n={n} k={w['k']} mean degree {w['deg']} p_out/p_in={w['ratio']:.4g}; "
            f"d={d}; Chebyshev order {order}; one step = one apply_filter of a device-resident block")


def run_reference(args, w, rank):
    """--impl reference: the CPU path on the host cores, rank 0 only."""
    if rank != 0:
        return
    from oracle import csc_oracle as O
    from oracle import native as ON
    codes, _ = make_graph_codes(w)
    n = w["n"]
    ip, ix, dv, _ = O.laplacian_csr(n, codes // n, codes % n, np.ones(codes.size))
    nnz = ix.size
    r = np.random.default_rng(11).standard_normal((n, w["d"])) / np.sqrt(w["d"])
    coeffs = O.step_coeffs(w["cutoff"], 2.0, w["order"])
    orders = 2
    for _ in range(args.warmup):
        cpu_filter_sample(ip, ix, dv, r, coeffs, orders)
    times = []
    cores = ON.num_threads()
    for _ in range(args.steps):
        dt, cores = cpu_filter_sample(ip, ix, dv, r, coeffs, orders)
        times.append(dt)
    t = float(np.mean(times))
    value = nnz * w["d"] * orders / t
    sample = f"{orders} of {w['order']} SpMM orders of apply_filter (C port, {cores} threads) per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(args.workload, w, n, w["d"], w["order"]), "n": n,
                   "nnz_L": int(nnz), "d": w["d"], "order": w["order"], "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def sweep_times(lib):
    buf = (ctypes.c_float * 4096)()
    cnt = ctypes.c_int(0)
    lib.csc_sweep_times(buf, 4096, ctypes.byref(cnt))
    return np.array(buf[: cnt.value], dtype=np.float64)


def timed_filter(lap, poly, blk, d, out, work, reps, lib):
    """(ms per filter by CUDA events on the launching stream, per-sweep ms)."""
    import torch
    from paper_1706_03591_b200.filters import filter_block
    filter_block(lap, poly, blk, d, out=out, work=work)
    torch.cuda.synchronize()
    lib.csc_sweep_timing(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        filter_block(lap, poly, blk, d, out=out, work=work)
    e1.record()
    torch.cuda.synchronize()
    lib.csc_sweep_timing(0)
    return e0.elapsed_time(e1) / reps, sweep_times(lib)


def run_cfg3_pipeline(lap, w, calls=3):
    """BASELINE configs[2] end to end through the public API: csc_assign
    (csc.py:87-108) on the cfg3 Laplacian — random signals d=128, eigencount
    bisection for lambda_100 (order 100), k-means k=100 (10 restarts) — ms per
    call (the first call warms plans and pools; the next `calls` are timed)."""
    import torch
    import paper_1706_03591_b200 as P
    k, d = w["k"], w["d"]
    fcfg = P.FilterConfig(order=w["order"])
    P.csc_assign(lap, k, d, fcfg, P.KmeansConfig(), seed=0)
    torch.cuda.synchronize()
    ms, diags = [], []
    for c in range(calls):
        t0 = time.perf_counter()
        a, diag = P.csc_assign(lap, k, d, fcfg, P.KmeansConfig(), seed=1 + c)
        torch.cuda.synchronize()
        ms.append((time.perf_counter() - t0) * 1e3)
        diags.append(diag)
    return {"workload": (f"configs[2] end to end: csc_assign(L, k={k}, d={d}, FilterConfig(order={w['order']}), "
                         f"KmeansConfig()) on the cfg3 graph (n={lap.n}): device signals, moment bisection "
                         f"for lambda_k, k-means k={k} x 10 restarts"),
            "ms_per_call": round(statistics.median(ms), 1), "ms_all": [round(v, 1) for v in ms],
            "lambda_k": diags[-1].lambda_k, "search_iters": diags[-1].search_iters,
            "matvecs_logical": diags[-1].matvecs}


def run_cfg4(hbm, lib):
    """BASELINE configs[3]: skewed-degree Chung-Lu graph, fp32 primary with an fp64 check."""
    import torch
    import paper_1706_03591_b200 as P
    from paper_1706_03591_b200 import generators as G
    from paper_1706_03591_b200._device import row_stride
    from paper_1706_03591_b200.signals import device_signals
    w = CFG4
    t0 = time.perf_counter()
    g, _ = G.chung_lu_sbm(w["n"], w["k"], w["deg"], w["exponent"], w["max_degree"], w["ratio"], seed=w["seed"])
    gen_s = time.perf_counter() - t0
    lap = P.laplacian(g)
    n, d, order, nnz = w["n"], w["d"], w["order"], lap.nnz
    poly = P.cheb_coeffs(w["cutoff"], lap.lambda_max_bound, order)
    x64 = device_signals(n, d, w["seed"])
    res = {"workload": (f"configs[3]: Chung-Lu / degree-corrected SBM n={n} k={w['k']} power-law exponent "
                        f"{w['exponent']} mean degree {w['deg']} max ~{int(w['max_degree'])} "
                        f"p_out/p_in={w['ratio']}; d={d}; Chebyshev order {order}"),
           "n": n, "nnz_L": int(nnz), "d": d, "order": order, "graph_gen_s": round(gen_s, 1)}
    outs = {}
    for prec, dt in (("fp32", torch.float32), ("fp64", torch.float64)):
        plan = lap.plan(1.0, dt)
        ld = row_stride(d, dt)
        blk = torch.zeros((n, ld), dtype=dt, device=x64.device)
        blk[:, :d].copy_(x64[:, :d])
        out = torch.empty_like(blk)
        work = torch.empty((2 * n, ld), dtype=dt, device=blk.device)
        ms, sw = timed_filter(lap, poly, blk, d, out, work, 2, lib)
        s = 8 if dt == torch.float64 else 4
        bm = b_min(n, nnz, d, s)
        sweep_ms = float(sw.mean())
        name, grid = last_launch(lib)
        entry = {"value": nnz * d * order / (ms / 1e3), "ms_per_step": ms, "sweep_ms_mean": sweep_ms,
                 "roofline_frac": bm / (sweep_ms / 1e3) / 1e9 / hbm, "bytes_min_per_launch": int(bm),
                 "schedule": "length_order" if plan.binned else "index_order",
                 "row_length_cv2": round(plan.len_cv2, 2), "long_rows": int(plan.n_long),
                 "kernel": name, "grid": grid}
        cap = traffic_capture("cfg4", prec)
        if cap is not None:
            entry["traffic"] = cap.get("dram_bytes_per_launch")
            entry["dram_frac"] = cap.get("dram_bytes_per_launch", 0) / (sweep_ms / 1e3) / 1e9 / hbm
            entry["traffic_source"] = cap["source"]
            entry["traffic_capture_matches"] = cap.get("kernel") == name and cap.get("grid") == grid
        res[prec] = entry
        outs[prec] = out[:, :d].double()
        del blk, work
    res["fp32_rel_frobenius_vs_fp64"] = float((outs["fp32"] - outs["fp64"]).norm() / outs["fp64"].norm())
    del outs, x64, lap
    torch.cuda.empty_cache()
    return res


def run_dynamic(args, rank):
    """ms per dynamic-CSC step on BASELINE configs[1]: SBM n=20k, k=20, mean degree 24,
    p_out/p_in=0.05, T=10 steps; each step moves 0.5% of nodes to another block
    (perturb_nodes) and then rewires 1% of edges (perturb_edges); d=80, p=0.5, m=60.
    The timed step includes merging that step's host insert/delete lists into the
    device edge set (Graph.apply_delta -> csc_edge_delta)."""
    import torch
    import paper_1706_03591_b200 as P
    from paper_1706_03591_b200 import generators as G
    n, k, d = 20000, 20, 80
    q1, q2 = G.sbm_probabilities(n, k, 24.0, 0.05)
    # the sequence from the device generators (8f-3); each step's lists are
    # handed to the timed step as host arrays, as a caller's would be
    g0, labels = G.planted_partition_device(n, k, 24.0, 0.05, seed=7)
    cur = g0
    steps = 10
    deltas = []
    for t in range(1, steps):  # nodes first, then edges
        dn, inn, labels = G.node_switch_device(cur, labels, k, q1, q2, 0.005, seed=200 + t)
        cur = cur.apply_delta(dn, inn)
        de, ie = G.edge_churn_device(cur, labels, q1, q2, 0.01, seed=100 + t)
        cur = cur.apply_delta(de, ie)
        deltas.append(tuple(x.cpu().numpy() for x in (dn, inn, de, ie)))
    cfg = P.DynamicConfig(k=k, d=d, p=0.5, filter=P.FilterConfig(order=60))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, state, diag0 = P.dynamic_init(g0, cfg, seed=rank)
    torch.cuda.synchronize()
    init_ms = (time.perf_counter() - t0) * 1e3
    ms, phases, refined = [], {}, 0
    g = g0
    for dn, inn, de, ie in deltas:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g = g.apply_delta(dn, inn).apply_delta(de, ie)  # host lists -> device merge
        t1 = time.perf_counter()
        _, state, diag = P.dynamic_step(state, g, cfg, timings=phases)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        ms.append((t2 - t0) * 1e3)
        phases["edge_delta"] = phases.get("edge_delta", 0.0) + (t1 - t0) * 1e3
        refined += diag.refined
    # one refined step: the communities split (k 20 -> 26 planted blocks), the
    # validation eigencount leaves the tolerance band and the cutoff is re-bisected
    g_split, _ = G.planted_partition_device(n, 26, 24.0, 0.05, seed=9)
    ph = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, _, diag_r = P.dynamic_step(state, g_split, cfg, timings=ph)
    torch.cuda.synchronize()
    refine_sample = {"ms": (time.perf_counter() - t0) * 1e3, "refined": bool(diag_r.refined),
                     "search_iters": diag_r.search_iters, "phase_ms": {k2: round(v, 3) for k2, v in ph.items()},
                     "graph": "SBM with 26 planted blocks (communities split); whole new edge set, not a delta"}
    out = {"workload": "configs[1] / cfg2: SBM n=20000 k=20 mean degree 24 p_out/p_in=0.05, T=10 (init + 9 steps), "
                       "per step 0.5% of nodes switch block then 1% of edges rewired; d=80 p=0.5 m=60, "
                       "k-means k=20 x 10 restarts; the step's insert/delete lists are merged on the device "
                       "inside the timed step", "ms_per_step": statistics.median(ms),
           "steps_timed": len(ms), "init_ms": init_ms, "refined_steps": refined,
           "phase_ms_total": {k2: round(v, 3) for k2, v in phases.items()},
           "refined_step": refine_sample}
    if rank == 0 and not args.no_cpu_baseline:
        # bounded CPU sample: one dynamic step through the oracle (C-port filter + numpy k-means)
        from oracle import csc_oracle as O
        from oracle import native as ON
        lap = P.laplacian(g)
        m = lap.matrix
        r = O.random_signals(n, 40, 1, scale_dim=d)
        coeffs = state.filter.coeffs
        t0 = time.perf_counter()
        fresh = ON.cheb_filter(m.indptr, m.indices, m.data, 2.0, coeffs, r)
        _ = O.count_from_block(fresh, 2.0)
        theta = np.concatenate([state.features.values[:, :40], fresh], axis=1)
        O.kmeans(theta, k, restarts=10, max_iters=100, tol=1e-6, seed=3)
        out["cpu_ms_per_step"] = (time.perf_counter() - t0) * 1e3
        out["cpu_sample"] = "1 step: C-port filter (all cores) + validation + numpy k-means (10 restarts)"
    return out


def run_dynamic_cfg5(args, rank, steps=4):
    """BASELINE configs[4] at p = 0.5 and 1% edge churn: planted partition n=2M,
    k=64, mean degree 20, p_out/p_in=0.05 (unspecified in BASELINE),
    d=96, m=80, fp64, k-means k=64 x 10 restarts. Timed step = device merge of
    the host insert/delete lists + dynamic_step (CSR rebuild, fresh signals,
    validation filter, (refine), Theta, k-means)."""
    import torch
    import paper_1706_03591_b200 as P
    from paper_1706_03591_b200 import generators as G
    w = WORKLOADS["cfg5"]
    n, k, d = w["n"], w["k"], w["d"]
    q1, q2 = G.sbm_probabilities(n, k, w["deg"], w["ratio"])
    t_gen = time.perf_counter()
    g, labels = G.planted_partition_device(n, k, w["deg"], w["ratio"], seed=w["seed"])  # device generators (8f-3)
    deltas, cur = [], g
    for s in range(steps):
        dl, il = G.edge_churn_device(cur, labels, q1, q2, 0.01, seed=50 + s)
        cur = cur.apply_delta(dl, il)
        deltas.append((dl.cpu().numpy(), il.cpu().numpy()))  # host lists for the timed merge
    gen_s = time.perf_counter() - t_gen
    cfg = P.DynamicConfig(k=k, d=d, p=0.5, filter=P.FilterConfig(order=w["order"]))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, state, diag0 = P.dynamic_init(g, cfg, seed=rank)
    torch.cuda.synchronize()
    init_ms = (time.perf_counter() - t0) * 1e3
    ms, phases, refined = [], {}, 0
    for dl, il in deltas:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g = g.apply_delta(dl, il)
        t1 = time.perf_counter()
        _, state, diag = P.dynamic_step(state, g, cfg, timings=phases)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        ms.append((t2 - t0) * 1e3)
        phases["edge_delta"] = phases.get("edge_delta", 0.0) + (t1 - t0) * 1e3
        refined += diag.refined
    return {"workload": (f"configs[4] / cfg5: planted partition n={n} k={k} mean degree {w['deg']} "
                         f"p_out/p_in={w['ratio']}; d={d} p=0.5 m={w['order']} fp64; 1% edge churn per step "
                         f"(insert/delete lists merged on the device inside the timed step); "
                         f"k-means k={k} x 10 restarts"),
            "ms_per_step": statistics.median(ms), "ms_all": [round(v, 1) for v in ms], "steps_timed": len(ms),
            "init_ms": init_ms, "init_search_iters": diag0.search_iters, "refined_steps": refined,
            "phase_ms_mean": {k2: round(v / len(ms), 2) for k2, v in phases.items()},
            "graph_and_churn_gen_s": round(gen_s, 2)}


def run_dynamic_cfg5_matrix(rank, steps=4, quality_steps=3):
    """BASELINE configs[4]'s sweep, sampled: churn {0.1%, 1%, 5%} at p = 0.5 and
    p {0, 0.25, 0.5} at 1% churn (p = 0.75 is rejected by the reference's
    DynamicConfig, dynamic.py:45-46), `steps` timed steps each (BASELINE: 20),
    the same device-generated graph sequence for every p of a churn level.
    Quality: ARI of the last step's labels against the planted partition, and
    the deviation versus p = 0 (ARI between the p run's and the p = 0 run's
    labels, and the difference of their planted-partition ARIs). BASELINE does
    not give p_out/p_in; at the timed ratio (0.05) the partition is at the
    detectability threshold, so the quality leg repeats p {0, 0.25, 0.5} at 1%
    churn on a detectable ratio (0.01) where the deviation is measurable."""
    import torch
    from sklearn.metrics import adjusted_rand_score as ari
    import paper_1706_03591_b200 as P
    from paper_1706_03591_b200 import generators as G
    w = WORKLOADS["cfg5"]
    n, k, d = w["n"], w["k"], w["d"]
    planted = np.repeat(np.arange(k), G.block_sizes(n, k))

    def run_cells(cells, ratio, nsteps, seed0):
        q1, q2 = G.sbm_probabilities(n, k, w["deg"], ratio)
        seqs, out, base_labels = {}, [], {}
        for churn, p in cells:
            if churn not in seqs:
                g, labels = G.planted_partition_device(n, k, w["deg"], ratio, seed=w["seed"])
                deltas, cur = [], g
                for s in range(nsteps):
                    dl, il = G.edge_churn_device(cur, labels, q1, q2, churn, seed=seed0 + s)
                    cur = cur.apply_delta(dl, il)
                    deltas.append((dl.cpu().numpy(), il.cpu().numpy()))
                seqs[churn] = (g, deltas)
            g, deltas = seqs[churn]
            cfg = P.DynamicConfig(k=k, d=d, p=p, filter=P.FilterConfig(order=w["order"]))
            _, state, _ = P.dynamic_init(g, cfg, seed=rank)
            ms, phases, gt = [], {}, g
            for dl, il in deltas:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                gt = gt.apply_delta(dl, il)
                a, state, _ = P.dynamic_step(state, gt, cfg, timings=phases)
                torch.cuda.synchronize()
                ms.append((time.perf_counter() - t0) * 1e3)
            cell = {"churn": churn, "p": p, "ms_per_step": round(statistics.median(ms), 1),
                    "ms_all": [round(v, 1) for v in ms],
                    "phase_ms_mean": {k2: round(v / len(ms), 1) for k2, v in phases.items()},
                    "ari_planted": round(float(ari(planted, a.labels)), 5)}
            if p == 0.0:
                base_labels[churn] = (a.labels, cell["ari_planted"])
            elif churn in base_labels:
                lab0, ari0 = base_labels[churn]
                cell["ari_vs_p0"] = round(float(ari(lab0, a.labels)), 5)
                cell["ari_planted_minus_p0"] = round(cell["ari_planted"] - ari0, 5)
            out.append(cell)
        return out

    cells = run_cells([(0.001, 0.5), (0.01, 0.0), (0.01, 0.25), (0.01, 0.5), (0.05, 0.5)], w["ratio"], steps, 500)
    res = {"workload": (f"configs[4] sweep sample: planted partition n={n} k={k} mean degree {w['deg']} "
                        f"p_out/p_in={w['ratio']}; d={d} m={w['order']} fp64; {steps} steps per cell "
                        f"(BASELINE: 20); same device-generated sequence for every p of a churn level; "
                        f"p=0.75 rejected by DynamicConfig (dynamic.py:45-46)"),
           "cells": cells,
           "note": ("p_out/p_in = 0.05 with mean degree 20 over 64 blocks sits near the detectability "
                    "threshold: ARI against the planted partition is ~0 for every p (DESIGN 4.6); "
                    "see quality for a detectable ratio")}
    if quality_steps > 0:
        qratio = 0.01
        res["quality"] = {"workload": (f"same shape at p_out/p_in={qratio} (detectable), 1% churn, "
                                       f"{quality_steps} steps per p; ARI of the last step's labels"),
                          "cells": run_cells([(0.01, 0.0), (0.01, 0.25), (0.01, 0.5)], qratio, quality_steps, 700)}
    return res


def e2e_calls(P, lap, poly, x_np, precision, calls):
    """Mean seconds per public apply_filter call (host numpy in, host numpy out)."""
    import torch
    for _ in range(2):  # steady state holds the previous result while the next call runs
        res = P.apply_filter(lap, poly, x_np, precision=precision)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(calls):
        res = P.apply_filter(lap, poly, x_np, precision=precision)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / calls, res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dynamic", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-cfg4", action="store_true")
    ap.add_argument("--no-cfg5", action="store_true")
    ap.add_argument("--no-cfg5-matrix", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    w = WORKLOADS[args.workload]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, w, rank)
        return

    import torch
    import torch.distributed as dist
    import paper_1706_03591_b200 as P
    from paper_1706_03591_b200 import _native
    from paper_1706_03591_b200 import signals as S
    from paper_1706_03591_b200._device import row_stride
    from paper_1706_03591_b200.filters import filter_block
    from paper_1706_03591_b200 import generators as G

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dtype = torch.float64 if args.precision == "fp64" else torch.float32
    n, d, order = w["n"], w["d"], w["order"]
    codes, _ = make_graph_codes(w)
    g = G.graph_from_codes(n, codes)
    lap = P.laplacian(g)
    nnz_L = lap.nnz
    plan = lap.plan(1.0, dtype)
    poly = P.cheb_coeffs(w["cutoff"], 2.0, order)
    rng = np.random.default_rng(1000 + rank)
    r_host = (rng.standard_normal((n, d)) / np.sqrt(d))
    dev = torch.device("cuda", local)
    ld = row_stride(d, dtype)
    blk = torch.zeros((n, ld), dtype=dtype, device=dev)
    blk[:, :d].copy_(torch.from_numpy(r_host).to(dev))
    out = torch.empty_like(blk)
    work = torch.empty((2 * n, ld), dtype=dtype, device=dev)

    def step():
        filter_block(lap, poly, blk, d, out=out, work=work)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    lib = _native.lib()
    lib.csc_sweep_timing(1)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        start.record()
        for _ in range(args.steps):
            step()
        end.record()
        torch.cuda.synchronize()
    lib.csc_sweep_timing(0)
    sweeps = sweep_times(lib)
    launch_name, launch_grid = last_launch(lib)
    ms = start.elapsed_time(end) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    units = nnz_L * d * order
    value = units * world / (ms / 1e3)

    # roofline of the dominant kernel (the fused sweep), algorithmic bytes per launch
    s = 8 if dtype == torch.float64 else 4
    bm = b_min(n, nnz_L, d, s)
    b_full = bm + 3 * n * d * s
    hbm, peak_kind = peaks()
    sweep_ms = float(sweeps.mean()) if sweeps.size else ms / order
    achieved = bm / (sweep_ms / 1e3) / 1e9
    cap = traffic_capture(args.workload, args.precision)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": cap.get("dram_bytes_per_launch") if cap else None, "peak_kind": peak_kind,
                "kernel": launch_name, "grid": launch_grid,
                "sweep_ms_mean": sweep_ms, "sweep_ms_median": float(np.median(sweeps)) if sweeps.size else None,
                "sweeps_timed": int(sweeps.size), "bytes_min_per_launch": int(bm),
                "bytes_full_per_launch": int(b_full), "frac_full": b_full / (sweep_ms / 1e3) / 1e9 / hbm,
                "sweep_share_of_step": float(sweeps.sum() / (ms * args.steps)) if sweeps.size else None,
                "nnz_M": int(plan.nnz), "schedule": "length_order" if plan.binned else "index_order"}
    if cap:
        roofline["traffic_source"] = cap["source"]
        roofline["traffic_capture"] = {k2: cap.get(k2) for k2 in ("kernel", "grid", "commit", "when")}
        roofline["traffic_capture_matches"] = cap.get("kernel") == launch_name and cap.get("grid") == launch_grid
        roofline["dram_frac"] = cap["dram_bytes_per_launch"] / (sweep_ms / 1e3) / 1e9 / hbm

    # end to end through the public API: host numpy in, host numpy out
    e2e = None
    if rank == 0 or world > 1:
        calls = max(5, args.steps)
        pinned = torch.from_numpy(r_host).pin_memory()
        e2e_s, res = e2e_calls(P, lap, poly, pinned.numpy(), args.precision, calls)
        e2e_pg, _ = e2e_calls(P, lap, poly, np.ascontiguousarray(r_host), args.precision, calls)
        if world > 1:
            t = torch.tensor([e2e_s, e2e_pg], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s, e2e_pg = (float(v) for v in t.tolist())
        e2e = {"value": units * world / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(n * d * 8),
               "d2h_bytes_per_step": int(res.nbytes), "ms_per_step": e2e_s * 1e3, "calls": calls,
               "api": "paper_1706_03591_b200.apply_filter(L, poly, numpy pinned) -> numpy",
               "pageable": {"value": units * world / e2e_pg, "ms_per_step": e2e_pg * 1e3, "calls": calls,
                            "api": "apply_filter(L, poly, ordinary numpy array) -> numpy (pinned staging "
                                   "ring, host threads)"}}
        del pinned, res

    # fp32 variant of the same workload, and configs[3]
    variants = {}
    if dtype == torch.float64 and not args.no_variants:
        blk32 = torch.zeros((n, row_stride(d, torch.float32)), dtype=torch.float32, device=dev)
        blk32[:, :d].copy_(blk[:, :d])
        out32 = torch.empty_like(blk32)
        work32 = torch.empty((2 * n, blk32.shape[1]), dtype=torch.float32, device=dev)
        lap.plan(1.0, torch.float32)
        ms32, sw32 = timed_filter(lap, poly, blk32, d, out32, work32, 2, lib)
        b32 = b_min(n, nnz_L, d, 4)
        variants["fp32"] = {"value": units * world / (ms32 / 1e3), "ms_per_step": ms32,
                            "roofline_frac": b32 / (float(sw32.mean()) / 1e3) / 1e9 / hbm,
                            "rel_frobenius_vs_fp64": float((out[:, :d] - out32[:, :d].double()).norm()
                                                           / out[:, :d].norm())}
        del blk32, out32, work32
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        m = lap.matrix
        dt, cores = cpu_filter_sample(m.indptr, m.indices, m.data, r_host, poly.coeffs, orders=2)
        cpu = {"value": nnz_L * d * 2 / dt, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"2 of {order} SpMM orders of apply_filter, C restatement on {cores} host threads "
                         f"(same graph and signals); {dt:.2f} s"}
        dt_ref = reference_scipy_sample(m, r_host, poly.coeffs, orders=2)
        if dt_ref is not None:
            cpu["reference_scipy"] = {
                "value": nnz_L * d * 2 / dt_ref, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": f"2 of {order} SpMM orders of the unmodified reference apply_filter "
                          f"(cscluster from baseline/_ref, SciPy csr_matvecs), same graph and signals, "
                          f"extrapolated per order; {dt_ref:.1f} s"}
    del blk, out, work
    torch.cuda.empty_cache()
    if dtype == torch.float64 and not args.no_variants and not args.no_pipeline:
        variants["cfg3_pipeline"] = run_cfg3_pipeline(lap, w)
    if dtype == torch.float64 and not args.no_variants and not args.no_cfg4:
        variants["cfg4"] = run_cfg4(hbm, lib)

    dyn = dyn5 = None
    if not args.no_dynamic:
        dyn = run_dynamic(args, rank)
        if not args.no_cfg5:
            del lap, plan
            torch.cuda.empty_cache()
            dyn5 = run_dynamic_cfg5(args, rank)
            if not args.no_cfg5_matrix:
                dyn5["matrix"] = run_dynamic_cfg5_matrix(rank)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64" if dtype == torch.float64 else "f32", "data": "synthetic",
            "config": {"workload": workload_desc(args.workload, w, n, d, order),
                       "n": n, "nnz_L": int(nnz_L), "d": d, "order": order, "precision": args.precision,
                       "l2": "inputs (n*d*8 B per block, 3 blocks) exceed the 126 MB L2; no flush",
                       "parallelism": f"column shards x{world}, no exchange"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(sweeps.size) if sweeps.size else int(order * args.steps),
            "clocks": clk.summary(),
            "rng": dict(S.RNG_STATS),
        }
        if variants:
            line["variants"] = variants
        if dyn is not None:
            line["dynamic"] = dyn
        if dyn5 is not None:
            line["dynamic_cfg5"] = dyn5
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
