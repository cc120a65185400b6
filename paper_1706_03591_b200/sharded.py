"""Column-sharded eigencount bisection and filtering across ranks.

The filter shards by columns with no halo exchange: each column's recurrence
is independent (filters.py:159-161) and every rank holds the full CSR. The
only exchange is the eigencount: the moments mu_q (or a per-probe energy) are
sums over columns, so one all-reduce(SUM) of 2m+1 doubles gives every rank
the global moments, every rank then runs the same host bisection and reaches
the same decisions, and each filters its own columns at the accepted cutoff.

The compute is injected (defaults: the GPU moment sweep and fused filter),
so the host protocol is tested on CPU with world_size 2 over gloo.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

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
