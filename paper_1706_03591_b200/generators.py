"""O(m) synthetic graph generators for the large BASELINE configurations.

The reference samplers are O(n^2) (one coin per vertex pair,
graphs.py:194-221; absent-pair enumeration, graphs.py:228-233) and cannot
produce configs 3-5 (n = 1M-4M). These produce graphs of the named shapes in
O(m) host work; they are input generators (not the measured hot path):

planted_partition  same model as sbm_generate (contiguous near-equal blocks,
                   q1 inside, q2 across; SbmParams' q1/q2 formula,
                   graphs.py:144-179): per block pair a Binomial edge count,
                   then that many distinct pairs drawn uniformly. Equal in
                   distribution to sbm_generate, not stream-identical.
chung_lu_sbm       degree-corrected SBM / Chung-Lu (config 4): power-law
                   expected degrees, endpoints drawn proportional to theta
                   inside the chosen block pair, duplicates and self-loops
                   discarded (the Poissonised Chung-Lu model).
edge_churn         per-step delete/insert code lists with perturb_edges
                   semantics (graphs.py:236-273): delete uniformly among
                   present edges, insert among absent pairs with probability
                   proportional to the model probability of the pair.

The same four models run on the GPU (csrc/generators.cu,
csc_gen_*): planted_partition_device, chung_lu_sbm_device,
edge_churn_device and node_switch_device keep the edge codes and the
delete/insert lists on the device (Graph.apply_delta takes device lists), with
O(k^2) host work only (the block-pair Binomial counts, the Chung-Lu pair
weights). The host versions above stay as the reference-style restatement
the device ones are tested against in distribution.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native
from ._device import ptr, require_cuda, stream
from .graphs import Graph


def _sorted_unique(codes: np.ndarray) -> np.ndarray:
    """np.unique for int64 codes by sort + adjacent dedup (numpy 2's hash-based
    unique is ~10x slower on tens of millions of codes); same result."""
    c = np.sort(codes)
    if c.size > 1:
        c = c[np.concatenate([[True], c[1:] != c[:-1]])]
    return c


def sbm_probabilities(n: int, k: int, s: float, e: float) -> tuple[float, float]:
    """q1, q2 with expected mean degree s and ratio e = q2/q1 (graphs.py:161-179)."""
    denom = (n / k - 1.0) + e * n * (k - 1) / k
    q1 = s / denom
    return min(q1, 1.0), min(e * q1, 1.0)


def block_sizes(n: int, k: int) -> np.ndarray:
    sizes = np.full(k, n // k, dtype=np.int64)
    sizes[: n % k] += 1
    return sizes


def _tri_unrank(idx: np.ndarray, s: int):
    """Index into the strict upper triangle of an s x s block -> (i, j), i < j."""
    # row i holds s-1-i pairs; offset(i) = i*(2s-i-1)/2
    i = np.floor((2 * s - 1 - np.sqrt((2 * s - 1) ** 2 - 8.0 * idx)) / 2).astype(np.int64)
    off = i * (2 * s - i - 1) // 2
    # fix floating-point rounding at row boundaries
    low = idx < off
    i[low] -= 1
    off = i * (2 * s - i - 1) // 2
    high = idx >= off + (s - 1 - i)
    i[high] += 1
    off = i * (2 * s - i - 1) // 2
    j = i + 1 + (idx - off)
    return i, j


def planted_partition_codes(n: int, k: int, q1: float, q2: float, seed=0) -> np.ndarray:
    """Sorted unique canonical codes lo*n+hi of a planted-partition graph."""
    rng = np.random.default_rng(seed)
    sizes = block_sizes(n, k)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    parts = []
    for a in range(k):
        sa, oa = int(sizes[a]), int(offs[a])
        npairs = sa * (sa - 1) // 2
        cnt = int(rng.binomial(npairs, q1)) if npairs else 0
        if cnt:
            idx = rng.choice(npairs, size=cnt, replace=False)
            i, j = _tri_unrank(idx.astype(np.int64), sa)
            parts.append((oa + i) * n + (oa + j))
        if q2 <= 0.0:
            continue
        # all blocks b > a at once: pairs (a, b) laid out back to back
        sb = sizes[a + 1:]
        if sb.size == 0:
            continue
        npair_b = sa * sb
        cnts = rng.binomial(npair_b, q2)
        tot = int(cnts.sum())
        if not tot:
            continue
        for b_rel in np.flatnonzero(cnts):
            c = int(cnts[b_rel])
            nb = int(npair_b[b_rel])
            idx = rng.choice(nb, size=c, replace=False)
            b = a + 1 + int(b_rel)
            sbb = int(sizes[b])
            i = oa + idx // sbb
            j = int(offs[b]) + idx % sbb
            parts.append(i * n + j)
    codes = np.concatenate(parts) if parts else np.empty(0, dtype=np.int64)
    codes.sort()
    return codes


def graph_from_codes(n: int, codes: np.ndarray) -> Graph:
    """Graph from sorted unique canonical codes (validated, no re-sort)."""
    codes = np.asarray(codes, dtype=np.int64)
    if codes.size > 1 and np.any(codes[1:] <= codes[:-1]):
        raise ValueError("codes must be strictly increasing")
    g = Graph.__new__(Graph)
    i, j = codes // n, codes % n
    if codes.size and (np.any(i >= j) or j.max() >= n or i.min() < 0):
        raise ValueError("codes must encode pairs i < j < n")
    g._init(int(n), i, j, np.ones(codes.size), None, int(codes.size))
    object.__setattr__(g, "_unit", True)
    return g


def planted_partition(n: int, k: int, mean_degree: float, ratio: float, seed=0) -> tuple[Graph, np.ndarray]:
    q1, q2 = sbm_probabilities(n, k, mean_degree, ratio)
    g = graph_from_codes(n, planted_partition_codes(n, k, q1, q2, seed))
    return g, np.repeat(np.arange(k, dtype=np.int64), block_sizes(n, k))


def chung_lu_sbm(n: int, k: int, mean_degree: float, exponent: float, max_degree: float,
                 ratio: float, seed=0) -> tuple[Graph, np.ndarray]:
    """Degree-corrected SBM with power-law expected degrees (config 4).

    theta_i proportional to (i + i0)^(-1/(exponent-1)), i0 chosen so the largest
    expected degree is ~max_degree at the requested mean; nodes are assigned to
    k contiguous blocks after a random permutation (so every block mixes hubs
    and leaves). The number of edge draws is Poisson(n * mean_degree / 2).
    """
    rng = np.random.default_rng(seed)
    gamma = 1.0 / (exponent - 1.0)
    # choose i0 so that theta_max / theta_mean = max_degree / mean_degree
    target = max_degree / mean_degree
    lo, hi = 1e-6, float(n)
    idx = np.arange(n, dtype=np.float64)
    for _ in range(60):
        i0 = np.sqrt(lo * hi)
        th = (idx + i0) ** -gamma
        r = th[0] / th.mean()
        if r > target:
            lo = i0
        else:
            hi = i0
    theta = (idx + i0) ** -gamma
    theta = theta / theta.mean() * mean_degree
    perm = rng.permutation(n)
    theta = theta[perm]
    sizes = block_sizes(n, k)
    blocks = np.repeat(np.arange(k), sizes)
    bw = np.array([theta[blocks == b].sum() for b in range(k)])
    # block-pair weights: inside w_in, across ratio * w_in
    pair_w = np.outer(bw, bw) * ratio
    pair_w[np.diag_indices(k)] = bw ** 2
    pair_w /= pair_w.sum()
    m_draw = rng.poisson(n * mean_degree / 2.0)
    # draw block pairs, then endpoints proportional to theta within blocks
    flat = rng.choice(k * k, size=m_draw, p=pair_w.ravel())
    ba, bb = flat // k, flat % k
    offs = np.concatenate([[0], np.cumsum(sizes)])
    cum = [np.cumsum(theta[offs[b]:offs[b + 1]]) for b in range(k)]
    ends_a = np.empty(m_draw, dtype=np.int64)
    ends_b = np.empty(m_draw, dtype=np.int64)
    # per-block index lists (stable sort = np.flatnonzero(side == b) for every b,
    # in one pass instead of 2k scans; same draws in the same order)
    groups = []
    for side in (ba, bb):
        order = np.argsort(side, kind="stable")
        bounds = np.concatenate([[0], np.cumsum(np.bincount(side, minlength=k))])
        groups.append((order, bounds))
    for b in range(k):
        for (order, bounds), out in zip(groups, (ends_a, ends_b)):
            sel = order[bounds[b]:bounds[b + 1]]
            if sel.size:
                u = rng.random(sel.size) * cum[b][-1]
                out[sel] = offs[b] + np.searchsorted(cum[b], u, side="right")
    ok = ends_a != ends_b
    lo_e = np.minimum(ends_a[ok], ends_b[ok])
    hi_e = np.maximum(ends_a[ok], ends_b[ok])
    codes = _sorted_unique(lo_e * n + hi_e)
    return graph_from_codes(n, codes), blocks


def edge_churn(codes: np.ndarray, n: int, labels: np.ndarray, q1: float, q2: float, fraction: float,
               seed=0) -> tuple[np.ndarray, np.ndarray]:
    """(deletes, inserts) sorted code lists redrawing round(fraction*m) edges.

    Deletes are uniform among present edges; inserts are drawn among absent
    pairs with probability proportional to q1 (same block) or q2 (different
    blocks), without replacement, as perturb_edges does (graphs.py:236-273);
    a just-deleted pair may be redrawn (it is then both deleted and inserted,
    which cancels: such pairs are dropped from both lists).
    """
    rng = np.random.default_rng(seed)
    m = codes.size
    count = int(round(fraction * m))
    if count == 0:
        return np.empty(0, np.int64), np.empty(0, np.int64)
    dels = np.sort(codes[rng.choice(m, size=count, replace=False)])
    kept = np.setdiff1d(codes, dels, assume_unique=True)
    k = int(labels.max()) + 1
    sizes = np.bincount(labels, minlength=k)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    # block members in label order (the identity for contiguous planted blocks;
    # labels stop being contiguous once nodes switch blocks)
    members = np.argsort(labels, kind="stable")
    # pair-class weights: same-block pairs and cross pairs
    n_in = float((sizes * (sizes - 1) // 2).sum())
    n_out = float(n) * (n - 1) / 2 - n_in
    w_in, w_out = q1 * n_in, q2 * n_out
    ins = np.empty(0, dtype=np.int64)
    need = count
    while need > 0:
        batch = int(need * 1.2) + 16
        inside = rng.random(batch) < w_in / (w_in + w_out)
        a = rng.integers(0, n, batch)
        b = np.empty(batch, dtype=np.int64)
        la = labels[a]
        bi = members[offs[la] + rng.integers(0, sizes[la])]
        b[inside] = bi[inside]
        bo = rng.integers(0, n, batch)
        b[~inside] = bo[~inside]
        ok = (a != b) & ((labels[a] == labels[b]) == inside)
        lo, hi = np.minimum(a[ok], b[ok]), np.maximum(a[ok], b[ok])
        cand = _sorted_unique(lo * n + hi)
        cand = cand[~np.isin(cand, kept, assume_unique=True)]
        cand = np.setdiff1d(cand, ins, assume_unique=True)
        rng.shuffle(cand)
        ins = np.concatenate([ins, cand[:need]])
        need = count - ins.size
    ins.sort()
    both = np.intersect1d(dels, ins, assume_unique=True)
    if both.size:
        dels = np.setdiff1d(dels, both, assume_unique=True)
        ins = np.setdiff1d(ins, both, assume_unique=True)
    return dels, ins


def node_switch(codes: np.ndarray, n: int, labels: np.ndarray, k: int, q1: float, q2: float,
                fraction: float, seed=0) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(deletes, inserts, new_labels) for reassigning round(fraction*n) nodes.

    perturb_nodes semantics (graphs.py:276-319): the selected nodes move to a
    uniformly drawn other block, all their incident edges are deleted, and
    every pair with a selected endpoint is then drawn once with the model
    probability under the new labels (q1 same block, q2 across). Equal in
    distribution, not stream-identical. O(count * n) host work (cfg2: 100 x 20k
    pairs); an edge deleted and redrawn is dropped from both lists.
    """
    if k < 2:
        raise ValueError("node reassignment needs k >= 2")
    rng = np.random.default_rng(seed)
    new_labels = np.asarray(labels, dtype=np.int64).copy()
    count = int(round(fraction * n))
    if count == 0:
        return np.empty(0, np.int64), np.empty(0, np.int64), new_labels
    sel = np.sort(rng.choice(n, size=count, replace=False))
    new_labels[sel] = (new_labels[sel] + rng.integers(1, k, size=count)) % k
    in_sel = np.zeros(n, dtype=bool)
    in_sel[sel] = True
    dels = codes[in_sel[codes // n] | in_sel[codes % n]]
    uu = np.repeat(sel, n)
    vv = np.tile(np.arange(n, dtype=np.int64), count)
    ok = uu != vv
    cand = _sorted_unique(np.minimum(uu[ok], vv[ok]) * n + np.maximum(uu[ok], vv[ok]))
    pi, pj = cand // n, cand % n
    prob = np.where(new_labels[pi] == new_labels[pj], q1, q2)
    ins = cand[rng.random(cand.size) < prob]
    both = np.intersect1d(dels, ins, assume_unique=True)
    if both.size:
        dels = np.setdiff1d(dels, both, assume_unique=True)
        ins = np.setdiff1d(ins, both, assume_unique=True)
    return dels, ins, new_labels


# ---------------------------------------------------------------------------
# Device generators (csrc/generators.cu)
# ---------------------------------------------------------------------------
def _device_seed(rng: np.random.Generator) -> int:
    return int(rng.integers(0, 2 ** 63, dtype=np.int64))


def _graph_from_device_codes(n: int, codes: torch.Tensor, m: int) -> Graph:
    g = Graph.__new__(Graph)
    g._init(int(n), None, None, None, codes[:m], int(m))
    object.__setattr__(g, "_unit", True)
    return g


def planted_pair_counts(n: int, k: int, q1: float, q2: float, rng: np.random.Generator) -> np.ndarray:
    """Binomial edge count per block pair (a <= b, row-major): Binomial(s_a (s_a - 1) / 2, q1)
    inside a block, Binomial(s_a s_b, q2) across — the planted partition's O(k^2) host part."""
    sizes = block_sizes(n, k)
    a, b = np.triu_indices(k)
    npairs = np.where(a == b, sizes[a] * (sizes[a] - 1) // 2, sizes[a] * sizes[b])
    return rng.binomial(npairs, np.where(a == b, q1, q2)).astype(np.int64)


def planted_partition_codes_device(n: int, k: int, q1: float, q2: float, seed=0) -> tuple[torch.Tensor, int]:
    """Sorted unique canonical codes of a planted-partition graph on the GPU (device tensor, m)."""
    dev = require_cuda()
    rng = np.random.default_rng(seed)
    counts = planted_pair_counts(n, k, q1, q2, rng)
    total = int(counts.sum())
    codes = torch.empty(max(total, 1), dtype=torch.int64, device=dev)
    m = ctypes.c_int64(0)
    _native.call("csc_gen_planted_partition", n, k, counts.ctypes.data, _device_seed(rng), ptr(codes),
                 codes.numel(), ctypes.byref(m), stream())
    return codes, int(m.value)


def planted_partition_device(n: int, k: int, mean_degree: float, ratio: float, seed=0) -> tuple[Graph, np.ndarray]:
    """planted_partition on the GPU: the graph's edge set never visits the host."""
    q1, q2 = sbm_probabilities(n, k, mean_degree, ratio)
    codes, m = planted_partition_codes_device(n, k, q1, q2, seed)
    return _graph_from_device_codes(n, codes, m), np.repeat(np.arange(k, dtype=np.int64), block_sizes(n, k))


def chung_lu_sbm_device(n: int, k: int, mean_degree: float, exponent: float, max_degree: float,
                        ratio: float, seed=0) -> tuple[Graph, np.ndarray]:
    """chung_lu_sbm on the GPU (same model and parameters): theta, its
    per-block cumulative sums and the edge draws on the device; the k x k
    block-pair weights and the Poisson draw count on the host."""
    dev = require_cuda()
    rng = np.random.default_rng(seed)
    gamma = 1.0 / (exponent - 1.0)
    target = max_degree / mean_degree
    idx = torch.arange(n, dtype=torch.float64, device=dev)
    lo, hi = 1e-6, float(n)
    for _ in range(60):  # i0 with theta_max / theta_mean = max_degree / mean_degree
        i0 = float(np.sqrt(lo * hi))
        th = (idx + i0) ** -gamma
        if float(th[0] / th.mean()) > target:
            lo = i0
        else:
            hi = i0
    theta = (idx + i0) ** -gamma
    theta = theta / theta.mean() * mean_degree
    perm = torch.from_numpy(rng.permutation(n)).to(dev)
    theta = theta[perm]
    sizes = block_sizes(n, k)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    cum = torch.empty_like(theta)
    bw = np.empty(k)
    for b in range(k):
        seg = torch.cumsum(theta[offs[b]:offs[b + 1]], 0)
        cum[offs[b]:offs[b + 1]] = seg
        bw[b] = float(seg[-1])
    pair_w = np.outer(bw, bw) * ratio
    pair_w[np.diag_indices(k)] = bw ** 2
    pair_cum = np.cumsum((pair_w / pair_w.sum()).ravel())
    m_draw = int(rng.poisson(n * mean_degree / 2.0))
    codes = torch.empty(max(m_draw, 1), dtype=torch.int64, device=dev)
    m = ctypes.c_int64(0)
    _native.call("csc_gen_chung_lu", n, k, ptr(cum), pair_cum.ctypes.data, m_draw, _device_seed(rng), ptr(codes),
                 codes.numel(), ctypes.byref(m), stream())
    return _graph_from_device_codes(n, codes, int(m.value)), np.repeat(np.arange(k, dtype=np.int64), sizes)


def _labels_dev(labels) -> torch.Tensor:
    if isinstance(labels, torch.Tensor):
        return labels.to(device=require_cuda(), dtype=torch.int32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(labels, dtype=np.int32)).to(require_cuda())


def edge_churn_device(g: Graph, labels, q1: float, q2: float, fraction: float,
                      seed=0) -> tuple[torch.Tensor, torch.Tensor]:
    """edge_churn on the GPU: (deletes, inserts) as sorted device code tensors."""
    dev = require_cuda()
    codes = g.device_codes()
    count = int(round(fraction * g.m))
    lab = _labels_dev(labels)
    k = int(lab.max().item()) + 1
    dels = torch.empty(max(count, 1), dtype=torch.int64, device=dev)
    ins = torch.empty(max(count, 1), dtype=torch.int64, device=dev)
    nd, ni = ctypes.c_int64(0), ctypes.c_int64(0)
    rng = np.random.default_rng(seed)
    _native.call("csc_gen_edge_churn", g.n, ptr(codes), g.m, ptr(lab), k, float(q1), float(q2), count,
                 _device_seed(rng), ptr(dels), ctypes.byref(nd), ptr(ins), ctypes.byref(ni), stream())
    return dels[:nd.value], ins[:ni.value]


def node_switch_device(g: Graph, labels, k: int, q1: float, q2: float, fraction: float,
                       seed=0) -> tuple[torch.Tensor, torch.Tensor, np.ndarray]:
    """node_switch on the GPU: (deletes, inserts) as sorted device code tensors, new labels (numpy)."""
    if k < 2:
        raise ValueError("node reassignment needs k >= 2")
    dev = require_cuda()
    codes = g.device_codes()
    count = int(round(fraction * g.n))
    lab = _labels_dev(labels).clone()
    dels = torch.empty(max(g.m, 1), dtype=torch.int64, device=dev)
    rng = np.random.default_rng(seed)
    dseed = _device_seed(rng)
    expected = count * g.n * max(q1, q2)
    cap = int(expected * 1.5 + 6 * np.sqrt(expected + 1) + 4096)
    nd, ni = ctypes.c_int64(0), ctypes.c_int64(0)
    while True:
        ins = torch.empty(cap, dtype=torch.int64, device=dev)
        lab_try = lab.clone()
        try:
            _native.call("csc_gen_node_switch", g.n, ptr(codes), g.m, ptr(lab_try), k, float(q1), float(q2), count,
                         dseed, ptr(dels), ctypes.byref(nd), ptr(ins), cap, ctypes.byref(ni), stream())
            break
        except ValueError as exc:  # CSC_ERR_CAPACITY: same draws with a larger buffer
            if "capacity" not in str(exc):
                raise
            cap *= 2
    return dels[:nd.value], ins[:ni.value], lab_try.cpu().numpy().astype(np.int64)
