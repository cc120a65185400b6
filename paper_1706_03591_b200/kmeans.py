"""Lloyd k-means with k-means++ seeding on the GPU (mirror of cscluster.kmeans).

Reference: /root/reference/pkg/src/cscluster/kmeans.py
  KmeansConfig  kmeans.py:17-28     Assignment   kmeans.py:31-51
  _kmeanspp_init kmeans.py:64-77    _lloyd       kmeans.py:88-117
  kmeans        kmeans.py:120-144   kmeans_cost  kmeans.py:147-157

The RNG stream is consumed on the host exactly as the reference does
(``integers(n)`` for the first centroid and the zero-mass fallback, one
``random()`` per D^2 draw, which is what ``Generator.choice(n, p=...)``
consumes), so the same seed picks the same centroid rows; distances, the
draw, assignment, repair, means and cost run in libcscb200. One 8-byte
device->host read per k-means++ draw and per Lloyd iteration carries the
values the reference branches on.
"""
from __future__ import annotations

import ctypes
import os
import threading
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from ._device import as_device_block, ptr, require_cuda, row_stride, stream
from .signals import FeatureMatrix, as_seed_sequence, block_nonfinite


@dataclass(frozen=True)
class KmeansConfig:
    restarts: int = 10
    max_iters: int = 100
    tol: float = 1e-6
    init: str = "kmeanspp"

    def __post_init__(self):
        if self.restarts < 1:
            raise ValueError("need at least one restart")
        if self.init != "kmeanspp":
            raise ValueError(f"unknown init {self.init!r}")


@dataclass(frozen=True, eq=False)
class Assignment:
    """Cluster labels plus sizes and the cost on the features it was solved on."""

    labels: np.ndarray
    cluster_sizes: np.ndarray
    feature_cost: float

    @property
    def n(self) -> int:
        return int(self.labels.size)

    @property
    def k(self) -> int:
        return int(self.cluster_sizes.size)

    def indicator(self) -> np.ndarray:
        """Dense n x k indicator X with entries 1/sqrt(s_j); X^T X = I."""
        x = np.zeros((self.n, self.k))
        x[np.arange(self.n), self.labels] = 1.0 / np.sqrt(self.cluster_sizes[self.labels])
        return x


class _Workspace:
    """Device buffers for one (features, k) problem, reused across restarts."""

    def __init__(self, blk: torch.Tensor, d: int, k: int):
        dev = blk.device
        self.blk, self.n, self.d, self.k = blk, blk.shape[0], d, k
        self.ld = blk.shape[1]
        self.ldc = row_stride(d)
        f64, i32 = torch.float64, torch.int32
        self.fnorm = torch.empty(self.n, dtype=f64, device=dev)
        self.cent = torch.zeros((k, self.ldc), dtype=f64, device=dev)
        self.cnorm = torch.empty(k, dtype=f64, device=dev)
        self.labels = torch.zeros(self.n, dtype=i32, device=dev)
        self.own = torch.empty(self.n, dtype=f64, device=dev)
        self.counts = torch.zeros(k, dtype=i32, device=dev)
        self.closest = torch.empty(self.n, dtype=f64, device=dev)
        self.nchunks = int(_native.lib().csc_kmeanspp_nchunks(self.n))
        self.chunk_sums = torch.empty(self.nchunks, dtype=f64, device=dev)
        self.scalars = torch.empty(2, dtype=f64, device=dev)
        self.idx = torch.empty(1, dtype=torch.int64, device=dev)
        _native.call("csc_kmeans_rownorms", ptr(blk), self.n, d, self.ld, ptr(self.fnorm), stream())

    # -- k-means++ (kmeans.py:64-77) ------------------------------------------
    def _pick(self, j: int, u: float = 0.0, fixed: int = -1):
        crow = self.cent[j]
        _native.call("csc_kmeanspp_pick", ptr(self.blk), self.n, self.d, self.ld, ptr(self.closest),
                     ptr(self.chunk_sums), self.nchunks, float(u), int(fixed), ptr(crow), ptr(self.idx),
                     stream())

    def _dist(self, j: int, first: bool):
        _native.call("csc_kmeanspp_dist", ptr(self.blk), self.n, self.d, self.ld, ptr(self.cent[j]),
                     ptr(self.closest), int(first), ptr(self.chunk_sums), self.nchunks, ptr(self.scalars),
                     stream())

    def kmeanspp(self, rng: np.random.Generator, record: list | None = None):
        n, k = self.n, self.k
        self._pick(0, fixed=int(rng.integers(n)))
        if record is not None:
            record.append(int(self.idx.item()))
        self._dist(0, True)
        for j in range(1, k):
            total = float(self.scalars[0].item())
            if total <= 0.0:
                self._pick(j, fixed=int(rng.integers(n)))
            else:
                self._pick(j, u=rng.random())
            if record is not None:
                record.append(int(self.idx.item()))
            if j < k - 1:
                self._dist(j, False)

    # -- Lloyd (kmeans.py:88-117) -------------------------------------------------
    def _plan(self):
        if getattr(self, "plan", None) is None:
            h = ctypes.c_void_p()
            _native.call("csc_kmeans_plan_create", self.n, self.d, self.ld, self.k, stream(), ctypes.byref(h))
            self.plan = h
        return self.plan

    def __del__(self):
        h = getattr(self, "plan", None)
        if h:
            try:
                _native.lib().csc_kmeans_plan_destroy(h)
            except Exception:
                pass
            self.plan = None

    def lloyd(self, max_iters: int, tol: float, history: list | None = None, pruned: bool = True):
        """Lloyd iterations from the seeds in self.cent; returns cost2 of the last one.

        pruned=True: bounds-pruned device iterations (csc_kmeans_iterate), cost
        by the centroid identity for the stop test and the exact difference
        form (kmeans.py:111) for the returned value.
        """
        if pruned:
            return self._lloyd_pruned(max_iters, tol, history)
        s = stream()
        n, d, k = self.n, self.d, self.k
        _native.call("csc_kmeans_rownorms", ptr(self.cent), k, d, self.ldc, ptr(self.cnorm), s)
        self.labels.zero_()
        prev = np.inf
        for _ in range(max_iters):
            _native.call("csc_kmeans_assign", ptr(self.blk), ptr(self.fnorm), n, d, self.ld, ptr(self.cent),
                         self.ldc, ptr(self.cnorm), k, ptr(self.labels), ptr(self.own), ptr(self.counts), s)
            _native.call("csc_kmeans_repair", ptr(self.labels), ptr(self.own), ptr(self.counts), n, k, s)
            _native.call("csc_kmeans_update", ptr(self.blk), ptr(self.labels), n, d, self.ld, k, ptr(self.cent),
                         self.ldc, ptr(self.cnorm), ptr(self.counts), s)
            _native.call("csc_kmeans_cost", ptr(self.blk), ptr(self.labels), ptr(self.cent), self.ldc, n, d,
                         self.ld, ptr(self.scalars[1:]), s)
            cost2 = float(self.scalars[1].item())
            if history is not None:
                history.append(np.sqrt(cost2))
            if np.isfinite(prev) and prev - cost2 <= tol * prev:
                prev = cost2
                break
            prev = cost2
        return prev

    def _lloyd_pruned(self, max_iters: int, tol: float, history: list | None):
        s = stream()
        n, d, k = self.n, self.d, self.k
        plan = self._plan()
        _native.call("csc_kmeans_rownorms", ptr(self.cent), k, d, self.ldc, ptr(self.cnorm), s)
        self.labels.zero_()
        prev = np.inf
        ran = False
        for it in range(max_iters):
            _native.call("csc_kmeans_iterate", plan, ptr(self.blk), ptr(self.fnorm), ptr(self.cent), self.ldc,
                         ptr(self.cnorm), ptr(self.labels), ptr(self.counts), int(it == 0), ptr(self.scalars[1:]),
                         s)
            ran = True
            cost2 = float(self.scalars[1].item())
            if history is not None:
                history.append(np.sqrt(cost2))
            if np.isfinite(prev) and prev - cost2 <= tol * prev:
                prev = cost2
                break
            prev = cost2
        if ran:  # returned cost in the reference's difference form
            _native.call("csc_kmeans_cost", ptr(self.blk), ptr(self.labels), ptr(self.cent), self.ldc, n, d,
                         self.ld, ptr(self.scalars[1:]), s)
            prev = float(self.scalars[1].item())
        return prev


class _Lane:
    """One concurrently running Lloyd restart: stream, plan (with its loop graph), buffers."""

    def __init__(self, pool, dev):
        n, d, ld, k = pool.n, pool.d, pool.ld, pool.k
        self.stream = torch.cuda.Stream(device=dev)
        self.ldc = row_stride(d)
        self.cent = torch.zeros((k, self.ldc), dtype=torch.float64, device=dev)
        self.cnorm = torch.empty(k, dtype=torch.float64, device=dev)
        self.labels = torch.zeros(n, dtype=torch.int32, device=dev)
        self.counts = torch.zeros(k, dtype=torch.int32, device=dev)
        self.out = torch.empty(2, dtype=torch.float64, device=dev)
        self.done = torch.cuda.Event()
        h = ctypes.c_void_p()
        _native.call("csc_kmeans_plan_create", n, d, ld, k, self.stream.cuda_stream, ctypes.byref(h))
        self.plan = h

    def __del__(self):
        h = getattr(self, "plan", None)
        if h:
            try:
                _native.lib().csc_kmeans_plan_destroy(h)
            except Exception:
                pass
            self.plan = None


class _LloydPool:
    """Persistent per-shape state so the Lloyd loop graphs are built once and reused."""

    MAX_LANES = 16

    def __init__(self, n, d, ld, k, dev):
        self.key = (dev.index, n, d, ld, k)
        self.n, self.d, self.ld, self.k = n, d, ld, k
        self.F = torch.zeros((n, ld), dtype=torch.float64, device=dev)
        self.ws = _Workspace(self.F, d, k)  # persistent row norms etc.: stable graph keys
        self.lanes = [_Lane(self, dev) for _ in range(self.MAX_LANES)]
        # FP32 screen of the assignment (same labels; csc_kmeans_plan_set_screen)
        self.screen = (os.environ.get("CSC_KMEANS_SCREEN", "1") != "0"
                       and bool(_native.lib().csc_kmeans_screen_supported(d, k)))
        if self.screen:
            self.ld32 = (d + 3) // 4 * 4
            self.F32 = torch.zeros((n, self.ld32), dtype=torch.float32, device=dev)
            self.fn32 = torch.empty(n, dtype=torch.float32, device=dev)
            for lane in self.lanes:
                _native.call("csc_kmeans_plan_set_screen", lane.plan, ptr(self.F32), self.ld32, ptr(self.fn32))

    def prepare(self, stream_handle):
        """Refresh the FP32 copy of F (after F changed)."""
        if self.screen:
            _native.call("csc_kmeans_screen_prepare", ptr(self.F), self.n, self.d, self.ld, ptr(self.F32),
                         self.ld32, ptr(self.fn32), stream_handle)


_LLOYD_POOL: _LloydPool | None = None  # the most recently used pool (tests / tools read it)
_LLOYD_POOLS: "OrderedDict[tuple, _LloydPool]" = OrderedDict()
POOL_SHAPES = 2  # per-shape pools kept (LRU): alternating shapes reuse their lanes and graphs


def _lloyd_pool(n, d, ld, k, dev) -> _LloydPool:
    global _LLOYD_POOL
    key = (dev.index, n, d, ld, k)
    pool = _LLOYD_POOLS.pop(key, None)
    if pool is None:
        while len(_LLOYD_POOLS) >= POOL_SHAPES:
            _LLOYD_POOLS.popitem(last=False)
        pool = _LloydPool(n, d, ld, k, dev)
    _LLOYD_POOLS[key] = pool
    _LLOYD_POOL = pool
    return pool


_POOL_LOCK = threading.Lock()  # the lanes / streams / buffers of the pool are shared state


def run_restarts(blk: torch.Tensor, d: int, k: int, cfg: KmeansConfig, children, draws=None,
                 fused: bool | None = None):
    """Thread-safe entry (the reference's kmeans is a pure function): one caller at a time.
    `draws` (optional) = kmeanspp_draws(children, n, k) made ahead of time.
    fused=None picks the single-launch fused Lloyd when the shape fits it
    (CSC_KMEANS_FUSED=0 disables), False forces the per-restart lanes."""
    n, ld = blk.shape
    if fused is None:
        fused = os.environ.get("CSC_KMEANS_FUSED", "1") != "0" and fused_supported(n, d, k, len(children),
                                                                                   cfg.max_iters)
    with _POOL_LOCK:
        if fused:
            try:
                return _run_fused(blk, d, k, cfg, children, draws)
            except _native.NativeError as exc:
                # the cooperative launch needs every block co-resident (one per
                # SM); with the GPU shared by other work it can be refused: the
                # per-restart lanes compute the same result
                if "cooperative" not in str(exc).lower():
                    raise
        return _run_restarts(blk, d, k, cfg, children, draws)


def fused_supported(n: int, d: int, k: int, restarts: int, max_iters: int) -> bool:
    """Whether csc_kmeans_fused_run takes this shape (features resident in shared memory)."""
    return bool(_native.lib().csc_kmeans_fused_supported(n, d, k, restarts, max_iters))


class _FusedState:
    """Persistent per-shape output buffers of the fused Lloyd path."""

    def __init__(self, n, d, ld, k, dev):
        self.key = (dev.index, n, d, ld, k)
        self.n, self.k, self.ldc, self.dev = n, k, row_stride(d), dev
        self.out = {}

    def outputs(self, R):
        """(labels R x n, packed bytes, cost R, iters R, seeds R x k x ldc, flags R): cost,
        iters and flags are views of one byte buffer, read back with one copy."""
        if R not in self.out:
            dev, n, k = self.dev, self.n, self.k
            packed = torch.empty(16 * R, dtype=torch.uint8, device=dev)
            self.out[R] = (torch.empty((R, n), dtype=torch.int32, device=dev), packed,
                           packed[:8 * R].view(torch.float64), packed[8 * R:12 * R].view(torch.int32),
                           torch.zeros((R, k, self.ldc), dtype=torch.float64, device=dev),
                           packed[12 * R:].view(torch.int32))
        return self.out[R]


_FUSED: _FusedState | None = None  # the most recently used output buffers
_FUSED_STATES: "OrderedDict[tuple, _FusedState]" = OrderedDict()
LAST_FUSED_ITERS: list[int] = []  # diagnostics: Lloyd iterations per restart of the last fused call


def _run_fused(blk: torch.Tensor, d: int, k: int, cfg: KmeansConfig, children, draws=None):
    """Every restart in one cooperative launch (csc_kmeans_fused_kpp_run): the
    k-means++ seeds from the restarts' host draws (integers(n), then k-1
    random(); kmeans.py:67-74) and all Lloyd runs in lock step, with the
    features resident in shared memory; best restart by the reference's rule
    (strictly smaller cost2, earliest on ties). A restart whose D^2 mass hit 0
    (the reference then draws integers(n)) is re-seeded on the sequential path
    and the launch repeated with explicit seeds. Returns (labels int64 numpy, cost2)."""
    global _FUSED
    dev = blk.device
    n, ld = blk.shape
    key = (dev.index, n, d, ld, k)
    st = _FUSED_STATES.pop(key, None)
    if st is None:
        while len(_FUSED_STATES) >= 4:
            _FUSED_STATES.popitem(last=False)
        st = _FusedState(n, d, ld, k, dev)
    _FUSED_STATES[key] = st
    _FUSED = st
    R = len(children)
    labels, packed, cost, iters, seeds, flags = _FUSED.outputs(R)
    ldc = _FUSED.ldc
    first, unif = draws if draws is not None else kmeanspp_draws(children, n, k)
    first = np.ascontiguousarray(first, dtype=np.int64)
    unif = np.ascontiguousarray(unif, dtype=np.float64)
    _native.call("csc_kmeans_fused_kpp_run", ptr(blk), n, d, ld, k, R, first.ctypes.data, unif.ctypes.data, ldc,
                 int(cfg.max_iters), float(cfg.tol), ptr(labels), ptr(cost), ptr(iters), ptr(seeds), ptr(flags),
                 stream())
    host = packed.cpu().numpy()  # one synchronising copy: costs, iterations, seeding flags
    costs, its, fl = host[:8 * R].view(np.float64), host[8 * R:12 * R].view(np.int32), host[12 * R:].view(np.int32)
    bad = [r for r in range(R) if fl[r] >= 0]
    if bad:  # zero D^2 mass (kmeans.py:70-72): sequential seeding for those restarts, explicit seeds
        ws = _Workspace(blk, d, k)
        for r in bad:
            ws.kmeanspp(np.random.default_rng(children[r]))
            seeds[r].copy_(ws.cent)
        _native.call("csc_kmeans_fused_run", ptr(blk), ptr(ws.fnorm), n, d, ld, k, R, ptr(seeds), ldc,
                     int(cfg.max_iters), float(cfg.tol), ptr(labels), ptr(cost), ptr(iters), stream())
        host = packed.cpu().numpy()
        costs, its = host[:8 * R].view(np.float64), host[8 * R:12 * R].view(np.int32)
    LAST_FUSED_ITERS[:] = [int(v) for v in its]
    best = 0
    for r in range(1, R):
        if costs[r] < costs[best]:
            best = r
    return labels[best].cpu().numpy().astype(np.int64), float(costs[best])


def _run_restarts(blk: torch.Tensor, d: int, k: int, cfg: KmeansConfig, children, draws=None):
    """Every restart: batched k-means++ seeds, then the Lloyd runs on concurrent lanes.

    Each lane runs iteration 1 and a device-resident loop graph
    (csc_kmeans_run); the best restart is chosen on the host with the
    reference's rule (strictly smaller cost2, earliest restart on ties).
    Returns (labels int64 numpy, cost2).
    """
    dev = blk.device
    n, ld = blk.shape
    pool = _lloyd_pool(n, d, ld, k, dev)
    cur = torch.cuda.current_stream()
    pool.F.copy_(blk)
    ws = pool.ws
    _native.call("csc_kmeans_rownorms", ptr(pool.F), n, d, ld, ptr(ws.fnorm), stream())
    pool.prepare(stream())
    # seeds are used right away; the rare zero-mass replay is checked at the
    # first host synchronisation and its restarts re-run (kmeans.py:70-72)
    seeds, bad_restarts, replay = batched_kmeanspp(ws, children, defer_check=True, draws=draws)
    R = len(children)
    costs: dict[int, float] = {}
    held: dict[int, int] = {}  # restart -> lane whose labels are still current

    serial = os.environ.get("CSC_KMEANS_SERIAL", "0") != "0"

    def run_wave(restarts):
        ready = torch.cuda.Event()
        ready.record(cur)
        for li, r in enumerate(restarts):
            lane = pool.lanes[li]
            st = pool.lanes[0].stream if serial else lane.stream  # serial: one stream, graphs back to back
            st.wait_event(ready)
            with torch.cuda.stream(st):
                lane.cent.copy_(seeds[r])
                _native.call("csc_kmeans_run", lane.plan, ptr(pool.F), ptr(ws.fnorm), ptr(lane.cent), lane.ldc,
                             ptr(lane.cnorm), ptr(lane.labels), ptr(lane.counts), int(cfg.max_iters),
                             float(cfg.tol), ptr(lane.out), None, st.cuda_stream)
                lane.done.record(st)
        for li in range(len(restarts)):
            cur.wait_event(pool.lanes[li].done)
        outs = torch.stack([pool.lanes[li].out[0] for li in range(len(restarts))]).cpu().numpy()
        held.clear()
        for li, r in enumerate(restarts):
            costs[r] = float(outs[li])
            held[r] = li

    best = None  # (cost2, restart); the reference keeps the earliest on ties (strict <)
    best_labels = None
    checked = False
    width = max(1, min(_LloydPool.MAX_LANES, int(os.environ.get("CSC_KMEANS_LANES", _LloydPool.MAX_LANES))))
    for w0 in range(0, R, width):
        wave = list(range(w0, min(R, w0 + width)))
        run_wave(wave)
        if not checked:  # the cost read above synchronised: the seeding flags are final
            checked = True
            redo = bad_restarts()
            if redo:
                KPP_REPLAYS[0] += len(redo)
                replay(redo)  # corrected seeds for every wave
                if any(r in wave for r in redo):
                    run_wave(wave)
        improved = False
        for r in wave:
            if best is None or costs[r] < best[0]:
                best = (costs[r], r)
                improved = True
        if improved:  # one labels copy per wave, of the best restart so far
            best_labels = pool.lanes[held[best[1]]].labels.cpu().numpy().astype(np.int64)
    return best_labels, best[0]


KPP_BATCH = 16  # restarts per batched k-means++ launch series (libcscb200 limit)
KPP_REPLAYS = [0]  # diagnostics: restarts re-seeded sequentially after a zero D^2 mass


def kpp_group(d: int) -> int:
    """Restarts per batched k-means++ series: their R x d centroids share one
    block's shared memory (<= ~200 KB of the 227 KB opt-in)"""
    return max(1, min(KPP_BATCH, (200 * 1024) // (8 * d + 32)))


def kmeanspp_draws(children, n: int, k: int):
    """Host RNG draws of every restart's k-means++ in the reference's order
    (kmeans.py:67-74): integers(n) for the first centroid, then k-1 random()
    (what Generator.choice(n, p) consumes). Returns (first int64[R], unif[R, k-1])."""
    rngs = [np.random.default_rng(c) for c in children]
    first = np.array([int(rng.integers(n)) for rng in rngs], dtype=np.int64)
    unif = np.ascontiguousarray(np.stack([rng.random(k - 1) for rng in rngs]) if k > 1
                                else np.zeros((len(rngs), 1)))
    return first, unif


def batched_kmeanspp(ws: _Workspace, children, defer_check: bool = False, draws=None):
    """k-means++ seeds of every restart: (restarts, k, ldc) on the GPU.

    Each restart's stream is drawn on the host in the reference's order
    (integers(n), then k-1 random(); kmeans.py:67-74) and the draws run in
    one batched device pass per centroid index. A restart that hits a zero
    D^2 mass (the reference then switches to integers(n)) is flagged by the
    device and replayed on the sequential path with a fresh generator.
    """
    n, k, R = ws.n, ws.k, len(children)
    seeds = torch.zeros((R, k, ws.ldc), dtype=torch.float64, device=ws.blk.device)
    per = kpp_group(ws.d)
    ngroups = (R + per - 1) // per
    flags = torch.empty((ngroups, per), dtype=torch.int32, device=ws.blk.device)
    all_first, all_unif = draws if draws is not None else kmeanspp_draws(children, n, k)
    for gidx, g0 in enumerate(range(0, R, per)):
        grp = list(range(g0, min(R, g0 + per)))
        first = np.ascontiguousarray(all_first[g0:g0 + len(grp)])
        unif = np.ascontiguousarray(all_unif[g0:g0 + len(grp)])
        _native.call("csc_kmeanspp_batch", ptr(ws.blk), n, ws.d, ws.ld, len(grp), k,
                     first.ctypes.data, unif.ctypes.data, ptr(seeds[g0]), ws.ldc, ptr(flags[gidx]), stream())

    def replay(bad_restarts):
        """Sequential k-means++ (fresh generator) for restarts whose D^2 mass hit 0."""
        for r in bad_restarts:
            ws.kmeanspp(np.random.default_rng(children[r]))
            seeds[r].copy_(ws.cent)

    def bad_restarts():
        fl = flags.cpu().numpy().reshape(-1)
        return [r for r in range(R) if fl[r] >= 0]

    if defer_check:  # the caller checks after launching work on the seeds
        return seeds, bad_restarts, replay
    replay(bad_restarts())
    return seeds


def _features_block(f):
    """Accept numpy / torch / FeatureMatrix features; validate like kmeans.py:127-134."""
    if isinstance(f, FeatureMatrix):
        return f.device_block(), f.d
    if isinstance(f, tuple):  # (padded block, d) from the internal pipeline
        return f
    if isinstance(f, torch.Tensor):
        if f.ndim != 2:
            raise ValueError("features must be a 2-d matrix")
        blk, d, _ = as_device_block(f)
        return blk, d
    f = np.asarray(f, dtype=np.float64)
    if f.ndim != 2:
        raise ValueError("features must be a 2-d matrix")
    if not np.all(np.isfinite(f)):
        raise ValueError("features must be finite")
    blk, d, _ = as_device_block(f)
    return blk, d


def kmeans(f, k: int, cfg: KmeansConfig | None = None, seed=0) -> Assignment:
    """Best of cfg.restarts Lloyd runs (k-means++ seeded); deterministic given seed.

    Each restart draws from its own spawned RNG stream; ties in cost keep the
    earliest restart (kmeans.py:136-144).
    """
    cfg = cfg or KmeansConfig()
    host = not isinstance(f, (FeatureMatrix, tuple, torch.Tensor))
    blk, d = _features_block(f)
    require_cuda()
    validated = isinstance(f, FeatureMatrix) and getattr(f, "_finite_checked", False)
    if not host and not validated and block_nonfinite(blk) != 0:
        raise ValueError("features must be finite")
    n = blk.shape[0]
    if not 1 <= k <= n:
        raise ValueError(f"need 1 <= k <= n, got k={k}, n={n}")
    children = as_seed_sequence(seed).spawn(cfg.restarts)
    return _kmeans_prepared(blk, d, k, cfg, children, None)


def _kmeans_prepared(blk, d: int, k: int, cfg: KmeansConfig, children, draws) -> Assignment:
    """kmeans() after validation, with the restarts' streams (and optionally their
    k-means++ draws) already made — the dynamic step draws them while the GPU
    filters."""
    labels, cost2 = run_restarts(blk, d, k, cfg, children, draws)
    sizes = np.bincount(labels, minlength=k)
    return Assignment(labels, sizes, float(np.sqrt(max(cost2, 0.0))))


def kmeans_cost(f, assignment: Assignment) -> float:
    """Cost ||F - X X^T F||_F of an existing assignment, in centroid form."""
    labels = np.asarray(assignment.labels)
    # the device kernels index shared memory and centroids by label: check the
    # range on the host first, with the reference's exception types
    # (np.bincount raises ValueError on negatives, np.add.at IndexError past k;
    # kmeans.py:80-85)
    if labels.ndim != 1 or (labels.size and not np.issubdtype(labels.dtype, np.integer)):
        raise ValueError("assignment labels must be a 1-D integer array")
    if labels.size and labels.min() < 0:
        raise ValueError("'list' argument must have no negative elements")
    if labels.size and labels.max() >= assignment.k:
        raise IndexError(f"index {int(labels.max())} is out of bounds for axis 0 with size {assignment.k}")
    blk, d = _features_block(f)
    if blk.shape[0] != assignment.n:
        raise ValueError("feature rows and assignment length differ")
    ws = _Workspace(blk, d, assignment.k)
    ws.labels.copy_(torch.from_numpy(labels.astype(np.int32)))
    s = stream()
    _native.call("csc_kmeans_update", ptr(blk), ptr(ws.labels), ws.n, d, ws.ld, ws.k, ptr(ws.cent), ws.ldc,
                 ptr(ws.cnorm), ptr(ws.counts), s)
    _native.call("csc_kmeans_cost", ptr(blk), ptr(ws.labels), ptr(ws.cent), ws.ldc, ws.n, d, ws.ld,
                 ptr(ws.scalars[1:]), s)
    return float(np.sqrt(ws.scalars[1].item()))
