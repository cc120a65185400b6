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
METRIC = "filtered nnz*d*order/s"
UNIT = "nnz*d*order/s"


def ncu_traffic(workload: str, precision: str):
    """DRAM bytes per sweep launch (read + write) from the committed ncu capture of
    this workload (profiles/r01_sweep_<workload>_<precision>_dram.csv), or None."""
    path = os.path.join(ROOT, "profiles", f"r01_sweep_{workload}_{precision}_dram.csv")
    if not os.path.exists(path):
        return None, None
    import csv
    per = {}
    with open(path) as fh:
        for r in csv.DictReader(ln for ln in fh if not ln.startswith("==")):
            if r["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[r["Metric Unit"]]
                per[r["ID"]] = per.get(r["ID"], 0.0) + float(r["Metric Value"].replace(",", "")) * scale
    if not per:
        return None, None
    return float(np.mean(list(per.values()))), os.path.relpath(path, ROOT)


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


def run_dynamic(args, rank):
    """ms per dynamic-CSC step on BASELINE configs[1]: SBM n=20k, k=20, mean degree 24,
    p_out/p_in=0.05, T=10 steps; each step moves 0.5% of nodes to another block
    (perturb_nodes) and then rewires 1% of edges (perturb_edges); d=80, p=0.5, m=60."""
    import torch
    import paper_1706_03591_b200 as P
    from paper_1706_03591_b200 import generators as G
    n, k, d = 20000, 20, 80
    q1, q2 = G.sbm_probabilities(n, k, 24.0, 0.05)
    codes = G.planted_partition_codes(n, k, q1, q2, 7)
    labels = np.repeat(np.arange(k), G.block_sizes(n, k))
    g = G.graph_from_codes(n, codes)
    graphs = [g]
    cur = codes
    steps = 10

    def applied(c, dl, il):
        return np.union1d(np.setdiff1d(c, dl, assume_unique=True), il)

    for t in range(1, steps):  # nodes first, then edges
        dn, inn, labels = G.node_switch(cur, n, labels, k, q1, q2, 0.005, seed=200 + t)
        cur = applied(cur, dn, inn)
        de, ie = G.edge_churn(cur, n, labels, q1, q2, 0.01, seed=100 + t)
        graphs.append(graphs[-1].apply_delta(dn, inn).apply_delta(de, ie))
        cur = applied(cur, de, ie)
    cfg = P.DynamicConfig(k=k, d=d, p=0.5, filter=P.FilterConfig(order=60))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, state, diag0 = P.dynamic_init(graphs[0], cfg, seed=rank)
    init_ms = (time.perf_counter() - t0) * 1e3
    ms, phases, refined = [], {}, 0
    for gt in graphs[1:]:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, state, diag = P.dynamic_step(state, gt, cfg, timings=phases)
        torch.cuda.synchronize()
        ms.append((time.perf_counter() - t0) * 1e3)
        refined += diag.refined
    out = {"workload": "configs[1] / cfg2: SBM n=20000 k=20 mean degree 24 p_out/p_in=0.05, T=10 (init + 9 steps), "
                       "per step 0.5% of nodes switch block then 1% of edges rewired; d=80 p=0.5 m=60, "
                       "k-means k=20 x 10 restarts", "ms_per_step": statistics.median(ms),
           "steps_timed": len(ms), "init_ms": init_ms, "refined_steps": refined,
           "phase_ms_total": {k2: round(v, 3) for k2, v in phases.items()}}
    if rank == 0 and not args.no_cpu_baseline:
        # bounded CPU sample: one dynamic step through the oracle (C-port filter + numpy k-means)
        from oracle import csc_oracle as O
        from oracle import native as ON
        lap = P.laplacian(graphs[1])
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
    buf = (__import__("ctypes").c_float * 4096)()
    cnt = __import__("ctypes").c_int(0)
    lib.csc_sweep_times(buf, 4096, __import__("ctypes").byref(cnt))
    sweeps = np.array(buf[: cnt.value], dtype=np.float64)
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
    b_min = 4 * (n + 1) + nnz_L * (4 + s) + nnz_L * d * s + n * d * s
    b_full = b_min + 3 * n * d * s
    hbm, peak_kind = peaks()
    sweep_ms = float(sweeps.mean()) if sweeps.size else ms / order
    achieved = b_min / (sweep_ms / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(args.workload, args.precision)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "traffic_source": traffic_src, "peak_kind": peak_kind,
                "kernel": "sweep_kernel (fused SpMM + recurrence)",
                "sweep_ms_mean": sweep_ms, "sweep_ms_median": float(np.median(sweeps)) if sweeps.size else None,
                "sweeps_timed": int(sweeps.size), "bytes_min_per_launch": int(b_min),
                "bytes_full_per_launch": int(b_full), "frac_full": b_full / (sweep_ms / 1e3) / 1e9 / hbm,
                "sweep_share_of_step": float(sweeps.sum() / (ms * args.steps)) if sweeps.size else None,
                "nnz_M": int(plan.nnz)}
    launches_per_step = order + (2 * order if plan.n_long else 0)

    # end to end through the public API: pinned host signals in, host features out
    e2e = None
    if rank == 0 or world > 1:
        pinned = torch.from_numpy(r_host).pin_memory()
        x_np = pinned.numpy()
        # warm-up in the same loop shape as the timed one (the previous result is
        # still alive during each call: steady state holds two pinned host outputs)
        for _ in range(2):
            res = P.apply_filter(lap, poly, x_np, precision=args.precision)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_steps = max(1, min(args.steps, 3))
        for _ in range(e2e_steps):
            res = P.apply_filter(lap, poly, x_np, precision=args.precision)
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        if world > 1:
            t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": units * world / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(n * d * 8),
               "d2h_bytes_per_step": int(res.nbytes), "ms_per_step": e2e_s * 1e3,
               "api": "paper_1706_03591_b200.apply_filter(L, poly, numpy pinned) -> numpy"}

    # fp32 variant of the same workload (reported separately; error in DESIGN.md)
    variants = {}
    if dtype == torch.float64 and not args.no_variants:
        blk32 = blk.to(torch.float32)
        ld32 = row_stride(d, torch.float32)
        if ld32 != blk32.shape[1]:
            b2 = torch.zeros((n, ld32), dtype=torch.float32, device=dev)
            b2[:, :d] = blk32[:, :d]
            blk32 = b2
        out32 = torch.empty_like(blk32)
        work32 = torch.empty((2 * n, blk32.shape[1]), dtype=torch.float32, device=dev)
        lap.plan(1.0, torch.float32)
        filter_block(lap, poly, blk32, d, out=out32, work=work32)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(2):
            filter_block(lap, poly, blk32, d, out=out32, work=work32)
        e1.record()
        torch.cuda.synchronize()
        ms32 = e0.elapsed_time(e1) / 2
        b32 = 4 * (n + 1) + nnz_L * 8 + nnz_L * d * 4 + n * d * 4
        variants["fp32"] = {"value": units * world / (ms32 / 1e3), "ms_per_step": ms32,
                            "roofline_frac": b32 / (ms32 / order / 1e3) / 1e9 / hbm,
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

    dyn = None
    if not args.no_dynamic:
        dyn = run_dynamic(args, rank)

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
            "gpu_launches": int(launches_per_step * args.steps), "clocks": clk.summary(),
        }
        if variants:
            line["variants"] = variants
        if dyn is not None:
            line["dynamic"] = dyn
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
