"""The column-sharded bisection with the product compute (sharded.py), two
ranks over gloo on one GPU: the ranks exchange only host scalars (the moment
vector, guard-band energies), so no kernel of one rank waits on the other.
Each rank filters its half of cfg1's signal columns on the GPU
(gpu_shard_fns: moment sweep + fused filter); both must reach the reference's
single-process cutoff and iteration count (golden), and the concatenated
features must equal the reference's features to 1e-10.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import paper_1706_03591_b200 as P
    from paper_1706_03591_b200.sharded import sharded_csc_features
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = np.load(os.path.join(GOLDEN, "cfg1.npz"))
        gr = P.Graph(int(g["g_n"]), g["g_i"], g["g_j"], g["g_w"])
        lap = P.laplacian(gr)
        sig_ss = np.random.SeedSequence(0).spawn(2)[0]  # the golden's signal stream (make_golden.py)
        out, (c0, c1), cut, iters, est = sharded_csc_features(lap, 10, 40, P.FilterConfig(order=50, max_iters=8),
                                                              seed=sig_ss)
        q.put((rank, cut, iters, est, c0, c1, out[:, :c1 - c0].cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_sharded_features_two_ranks_product_compute(cuda_ok):
    g = np.load(os.path.join(GOLDEN, "cfg1.npz"))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1] == float(g["cutoff"])
    assert res[0][2] == res[1][2] == int(g["iters"])
    assert abs(res[0][3] - float(g["est"])) <= 1e-10 * float(g["est"])
    feats = np.concatenate([res[0][6], res[1][6]], axis=1)
    ref = g["features"]
    assert np.linalg.norm(feats - ref) <= 1e-10 * np.linalg.norm(ref)
