"""Column-sharded eigencount bisection and filtering across ranks.

The filter shards by columns with no halo exchange: each column's recurrence
is independent (filters.py:159-161) and every rank holds the full CSR. The
only exchange is the eigencount: the moments mu_q (or a per-probe energy) are
sums over columns, so one all-reduce(SUM) of 2m+1 doubles gives every rank
the global moments, every rank then runs the same host bisection and reaches
the same decisions, and each filters its own columns at the accepted cutoff.

The compute is injected (defaults: the GPU moment sweep and fused filter),
so the host protocol is tested on CPU with world_size 2 over gloo; the public
entry sharded_csc_features (csc_features, csc.py:72-84, over column shards)
runs it with the product compute (tests/test_gpu_sharded.py: two gloo ranks
on one GPU reach the single-process cutoff, iterations and features).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _native
from ._device import ptr, require_cuda, row_stride, stream
from .filters import (EigencountSearchError, FilterConfig, MOMENT_GUARD, cheb_coeffs,
                      moment_energy)


def shard_columns(d: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous column range [c0, c1) of rank `rank`."""
    base, extra = divmod(d, world)
    c0 = rank * base + min(rank, extra)
    return c0, c0 + base + (1 if rank < extra else 0)


def allreduce_sum(values: np.ndarray, group=None) -> np.ndarray:
    """Sum a small float64 vector over ranks (device tensor under nccl)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return np.asarray(values, dtype=np.float64)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.as_tensor(np.asarray(values, dtype=np.float64), device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy()


def sharded_search_cutoff(k: int, interval, lambda_max: float, cfg: FilterConfig, moments_fn, filter_fn,
                          count_scale: float = 1.0, group=None):
    """Moment bisection over column shards (same decisions as filters.py:233-255).

    moments_fn(m) -> this rank's mu (2m+1,) over its columns;
    filter_fn(coeffs) -> (this rank's filtered block, this rank's energy).
    Returns (cutoff, local filtered block, coeffs, iterations, global estimate).
    """
    lo, hi = float(interval[0]), float(interval[1])
    if not 0.0 <= lo < hi <= lambda_max + 1e-12:
        raise ValueError("search interval must satisfy 0 <= lo < hi <= lambda_max_bound")
    mu = None
    mid = est = None
    for it in range(1, cfg.max_iters + 1):
        mid = 0.5 * (lo + hi)
        poly = cheb_coeffs(mid, lambda_max, cfg.order, damping=cfg.damping, response=cfg.response,
                           sigmoid_sharpness=cfg.sigmoid_sharpness)
        if mu is None:
            mu = allreduce_sum(moments_fn(poly.coeffs.size - 1), group)
        est = moment_energy(mu, poly.coeffs) * count_scale
        out = None
        thresholds = (k - cfg.count_tol * k, k + cfg.count_tol * k, float(k))
        if min(abs(est - t) for t in thresholds) <= MOMENT_GUARD * max(1.0, abs(k)):
            out, e_local = filter_fn(poly.coeffs)
            est = float(allreduce_sum(np.array([e_local]), group)[0]) * count_scale
        accept = abs(est - k) <= cfg.count_tol * k
        if not accept:
            if est > k:
                hi = mid
            else:
                lo = mid
            accept = hi - lo < cfg.width_tol
        if accept:
            if out is None:
                out, e_local = filter_fn(poly.coeffs)
                est = float(allreduce_sum(np.array([e_local]), group)[0]) * count_scale
            return mid, out, poly.coeffs, it, est
    raise EigencountSearchError(
        f"no acceptable cutoff after {cfg.max_iters} probes (last cutoff {mid:.6g}, estimate {est:.4g}, "
        f"target {k})", last_cutoff=mid, last_estimate=est, iterations=cfg.max_iters)


def gpu_shard_fns(L, blk, d: int, lambda_max: float):
    """The product compute for one rank's device block (moment sweep + fused filter)."""
    from .filters import FilterPoly, block_moments, filter_block

    def moments_fn(m):
        return block_moments(L, blk, d, m, lambda_max)

    def filter_fn(coeffs):
        poly = FilterPoly(len(coeffs) - 1, np.asarray(coeffs), 0.0, lambda_max, "")
        out, s = filter_block(L, poly, blk, d, None, want_sumsq=True)
        return out, float(s.item())

    return moments_fn, filter_fn


def shard_signals(n: int, d: int, c0: int, c1: int, seed=0) -> torch.Tensor:
    """Columns [c0, c1) of random_signals(n, d, seed) (signals.py:16-37) as a
    padded (n, ld) float64 device block: the same per-column PCG64 streams the
    single-process draw uses (numpy's SeedSequence children c0..c1-1), drawn
    on the GPU; flagged columns are redrawn with the exact host generator."""
    from .signals import as_seed_sequence, child_states
    if not 0 <= c0 < c1 <= d:
        raise ValueError("need 0 <= c0 < c1 <= d")
    ss = as_seed_sequence(seed)
    base = int(ss.n_children_spawned)
    states = np.ascontiguousarray(child_states(ss, d)[c0:c1])
    nc = c1 - c0
    blk = torch.zeros((n, row_stride(nc)), dtype=torch.float64, device=require_cuda())
    bad = np.zeros(nc, dtype=np.int32)
    sigma = 1.0 / np.sqrt(d)
    _native.call("csc_normal_columns", states.ctypes.data, nc, n, sigma, ptr(blk), blk.shape[1], 0,
                 bad.ctypes.data, stream())
    for c in np.flatnonzero(bad):
        child = np.random.SeedSequence(ss.entropy, spawn_key=tuple(ss.spawn_key) + (base + c0 + int(c),),
                                       pool_size=ss.pool_size)
        blk[:, c].copy_(torch.from_numpy(np.random.default_rng(child).standard_normal(n) * sigma + 0.0))
    return blk


def sharded_csc_features(L, k: int, d: int, filter_cfg: FilterConfig | None = None, seed=0, group=None):
    """csc_features (csc.py:72-84) over column shards: this rank draws and
    filters columns shard_columns(d, world, rank) of the same signal block,
    the ranks agree on the cutoff through one all-reduce of the 2m+1 moments
    (and of the energy at guard-band probes), and each returns its slice of
    the features. Returns (local features (n, ld) device block, (c0, c1),
    cutoff, iterations, global estimate)."""
    cfg = filter_cfg or FilterConfig()
    if not 1 <= k < L.n:
        raise ValueError(f"need 1 <= k < n, got k={k}, n={L.n}")
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    c0, c1 = shard_columns(d, world, rank)
    blk = shard_signals(L.n, d, c0, c1, seed)
    moments_fn, filter_fn = gpu_shard_fns(L, blk, c1 - c0, L.lambda_max_bound)
    cutoff, out, _, iters, est = sharded_search_cutoff(k, (0.0, L.lambda_max_bound), L.lambda_max_bound, cfg,
                                                       moments_fn, filter_fn, 1.0, group)
    return out, (c0, c1), cutoff, iters, est
