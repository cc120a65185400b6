"""N>1 path on CPU: column-sharded moment bisection over gloo, world_size 2.

Each rank holds half of cfg1's signal columns; the oracle supplies the
per-rank compute (the GPU kernels are injected the same way in the product).
The sharded run must reach the reference's single-process cutoff/iterations
and, concatenated, its features.
"""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from conftest import GOLDEN


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from oracle import csc_oracle as O
    from paper_1706_03591_b200.filters import FilterConfig
    from paper_1706_03591_b200.sharded import shard_columns, sharded_search_cutoff
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = np.load(os.path.join(GOLDEN, "cfg1.npz"))
        ip, ix, dv = g["L_indptr"], g["L_indices"], g["L_data"]
        c0, c1 = shard_columns(40, world, rank)
        x = g["R"][:, c0:c1]

        def moments_fn(m):
            return O.moments(ip, ix, dv, 2.0, x, m)

        def filter_fn(coeffs):
            out = O.apply_filter(ip, ix, dv, 2.0, coeffs, x)
            return out, float((out ** 2).sum())

        cfg = FilterConfig(order=50, max_iters=8)
        cut, out, coeffs, iters, est = sharded_search_cutoff(10, (0.0, 2.0), 2.0, cfg, moments_fn, filter_fn)
        q.put((rank, cut, iters, est, c0, c1, out))
    finally:
        dist.destroy_process_group()


def test_sharded_bisection_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = np.load(os.path.join(GOLDEN, "cfg1.npz"))
    res.sort()
    assert res[0][1] == res[1][1] == float(g["cutoff"])
    assert res[0][2] == res[1][2] == int(g["iters"])
    assert abs(res[0][3] - float(g["est"])) <= 1e-10 * float(g["est"])
    feats = np.concatenate([res[0][6], res[1][6]], axis=1)
    assert np.array_equal(feats, g["features"])


def test_shard_columns_cover():
    from paper_1706_03591_b200.sharded import shard_columns
    for d in (1, 7, 40, 128):
        for w in (1, 2, 3, 8):
            ranges = [shard_columns(d, w, r) for r in range(w)]
            assert ranges[0][0] == 0 and ranges[-1][1] == d
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
