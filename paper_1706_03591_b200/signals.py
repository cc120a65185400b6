"""Random probe signals and device-resident feature blocks (mirror of cscluster.signals).

Reference: /root/reference/pkg/src/cscluster/signals.py
  as_seed_sequence  signals.py:9-13
  random_signals    signals.py:16-37  (same numpy PCG64/SeedSequence streams,
                                        bit-identical values)
  FeatureMatrix     signals.py:40-87  (same fields and checks; the values live
                                        on the GPU as a padded row-major block
                                        and are copied to the host on access)
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import _native
from ._device import download_block, ptr, require_cuda, row_stride, stream, upload_block


def as_seed_sequence(seed) -> np.random.SeedSequence:
    """Coerce an integer seed (or pass through a SeedSequence) for stream spawning."""
    if isinstance(seed, np.random.SeedSequence):
        return seed
    return np.random.SeedSequence(seed)


_POOL = None


def _pool():
    global _POOL
    if _POOL is None:
        _POOL = ThreadPoolExecutor(max_workers=max(1, min(32, os.cpu_count() or 1)),
                                   thread_name_prefix="csc-rng")
    return _POOL


def signal_columns(n: int, d: int, seed=0, scale_dim: int | None = None) -> np.ndarray:
    """The random block column-major: (d, n), row c = column c of random_signals.

    Column c is sigma * standard_normal(n) from default_rng(SeedSequence(seed)
    .spawn(d)[c]) -- the same draws as the reference's normal(0.0, sigma, n)
    and the same bits (0.0 + sigma*z, signals.py:34-37). Columns are
    independent streams, generated in a thread pool (numpy releases the GIL).
    """
    if d < 1:
        raise ValueError("need at least one signal column")
    if n < 1:
        raise ValueError("need at least one node")
    dim = d if scale_dim is None else int(scale_dim)
    if dim < 1:
        raise ValueError("scale_dim must be positive")
    sigma = 1.0 / np.sqrt(dim)
    children = as_seed_sequence(seed).spawn(d)
    cols = np.empty((d, n))

    def fill(c):
        row = cols[c]
        np.random.default_rng(children[c]).standard_normal(size=n, out=row)
        row *= sigma
        row += 0.0

    if n * d >= 1 << 20 and d > 1:
        list(_pool().map(fill, range(d)))
    else:
        for c in range(d):
            fill(c)
    return cols


def random_signals(n: int, d: int, seed=0, scale_dim: int | None = None) -> np.ndarray:
    """n x d i.i.d. N(0, 1/scale_dim); column c from SeedSequence(seed).spawn(d)[c]."""
    return np.ascontiguousarray(signal_columns(n, d, seed, scale_dim).T)


# "device": PCG64 + ziggurat on the GPU (csc_normal_columns); "host": numpy in
# a thread pool + H2D (bit-exact by construction). CSC_RNG=host selects the latter.
RNG_MODE = os.environ.get("CSC_RNG", "device")
# columns the device generator flagged (chunk boundaries that did not agree)
# and the host regenerated; reported by bench.py, asserted zero in the tests
RNG_STATS = {"device_columns": 0, "redrawn_columns": 0}


def _u32_words(x) -> list[int]:
    """numpy's SeedSequence word coercion (bit_generator.pyx _coerce_to_uint32_array)
    for integers and (nested) integer sequences: little-endian 32-bit words,
    [0] for zero."""
    if isinstance(x, np.ndarray) and x.dtype == np.uint32:
        return [int(v) for v in x]
    if isinstance(x, (int, np.integer)):
        v = int(x)
        if v < 0:
            raise ValueError("expected non-negative integer")
        if v == 0:
            return [0]
        words = []
        while v > 0:
            words.append(v & 0xFFFFFFFF)
            v >>= 32
        return words
    out: list[int] = []
    for v in x:
        out.extend(_u32_words(v))
    return out


def child_states(ss: np.random.SeedSequence, d: int) -> np.ndarray:
    """column_states(ss.spawn(d)) computed in the library (csc_seed_states) without
    building the children: (d, 4) uint64 (state lo, hi, inc lo, hi) of
    PCG64(child) for children ss.n_children_spawned .. + d - 1. Does not advance ss."""
    run = np.ascontiguousarray(_u32_words(ss.entropy), dtype=np.uint32)
    key = np.ascontiguousarray(_u32_words(ss.spawn_key), dtype=np.uint32)
    out = np.empty((d, 4), dtype=np.uint64)
    _native.call("csc_seed_states", run.ctypes.data, run.size, key.ctypes.data, key.size,
                 int(ss.n_children_spawned), d, int(ss.pool_size), out.ctypes.data)
    return out


def column_states(children) -> np.ndarray:
    """Initial PCG64 (state, inc) of each child stream as 4 uint64 words per column."""
    words = np.empty((len(children), 4), dtype=np.uint64)
    mask = (1 << 64) - 1
    for c, child in enumerate(children):
        st = np.random.PCG64(child).state["state"]
        s, inc = int(st["state"]), int(st["inc"])
        words[c] = (s & mask, s >> 64, inc & mask, inc >> 64)
    return words


def device_signals(n: int, d: int, seed=0, scale_dim: int | None = None, mode: str | None = None,
                   advance: bool = True, defer: bool = False):
    """random_signals as a padded (n, ld) float64 device block.

    Device mode draws numpy's exact PCG64 streams and ziggurat on the GPU;
    columns the generator flags are redrawn on the host (the exact path). The
    per-column PCG64 states come from the library's SeedSequence restatement;
    a caller's SeedSequence is advanced by d children as ss.spawn(d) would
    (advance=False skips that for internal, never-reused children).
    defer=True (device mode): returns (block, fix) without synchronising;
    fix() reads the device flags, redraws flagged columns on the host and
    returns whether it changed any (the caller then recomputes what it built
    from the block).
    """
    if d < 1:
        raise ValueError("need at least one signal column")
    if n < 1:
        raise ValueError("need at least one node")
    dim = d if scale_dim is None else int(scale_dim)
    if dim < 1:
        raise ValueError("scale_dim must be positive")
    dev = require_cuda()
    blk = torch.zeros((n, row_stride(d)), dtype=torch.float64, device=dev)
    if (mode or RNG_MODE) == "device":
        ss = as_seed_sequence(seed)
        base = int(ss.n_children_spawned)
        states = child_states(ss, d)
        if advance and ss is seed:  # the caller's SeedSequence moves on exactly as in signal_columns
            ss.spawn(d)
        sigma = 1.0 / np.sqrt(dim)

        RNG_STATS["device_columns"] += d

        def redraw(bad):  # flagged columns: the exact host generator
            RNG_STATS["redrawn_columns"] += int(np.count_nonzero(bad))
            for c in np.flatnonzero(bad):
                child = np.random.SeedSequence(ss.entropy, spawn_key=tuple(ss.spawn_key) + (base + int(c),),
                                               pool_size=ss.pool_size)
                z = np.random.default_rng(child).standard_normal(n) * sigma + 0.0
                blk[:, c].copy_(torch.from_numpy(z))
            return bool(np.any(bad))

        if defer:  # no synchronisation here: the caller runs fix() at its next one
            bad_dev = torch.empty(d, dtype=torch.int32, device=dev)
            _native.call("csc_normal_columns_async", states.ctypes.data, d, n, float(sigma), ptr(blk),
                         blk.shape[1], 0, ptr(bad_dev), stream())
            return blk, lambda: redraw(bad_dev.cpu().numpy())
        bad = np.zeros(d, dtype=np.int32)
        _native.call("csc_normal_columns", states.ctypes.data, d, n, float(sigma), ptr(blk), blk.shape[1], 0,
                     bad.ctypes.data, stream())
        redraw(bad)
        return blk
    cols = torch.from_numpy(signal_columns(n, d, seed, scale_dim))
    blk[:, :d].copy_(cols.to(dev).t())
    return (blk, lambda: False) if defer else blk


def block_nonfinite(blk: torch.Tensor) -> int:
    """Count of non-finite entries of a device block (one sync)."""
    s = torch.empty(1, dtype=torch.float64, device=blk.device)
    bad = torch.zeros(1, dtype=torch.int64, device=blk.device)
    code = _native.CSC_F64 if blk.dtype == torch.float64 else _native.CSC_F32
    _native.call("csc_sumsq", ptr(blk), blk.numel(), code, ptr(s), ptr(bad), stream())
    return int(bad.item())


def gather_columns(src: torch.Tensor, cols, dst: torch.Tensor, col0: int = 0) -> None:
    """dst[:, col0 + j] = src[:, cols[j]] (float64 blocks) on the GPU."""
    cols_t = torch.as_tensor(np.asarray(cols, dtype=np.int64)).to(src.device)
    if cols_t.numel() == 0:
        return
    _native.call("csc_gather_columns", ptr(src), src.shape[0], src.shape[1], ptr(cols_t), cols_t.numel(),
                 ptr(dst), dst.shape[1], col0, stream())


class FeatureMatrix:
    """Block of filtered signals with per-column provenance tags.

    ``step_tags[c]`` records the time step whose graph filtered column c and
    ``stream_tags[c]`` the RNG stream index within that step's draw. Values are
    float64 and must be finite (ValueError otherwise), as in signals.py:53-62.
    """

    def __init__(self, values, step_tags, stream_tags):
        if isinstance(values, torch.Tensor):
            if values.ndim != 2:
                raise ValueError("feature values must be a 2-d matrix")
            n, d = values.shape
            blk = torch.zeros((n, row_stride(d)), dtype=torch.float64, device=require_cuda())
            blk[:, :d].copy_(values)
            self._set(blk, d, None, step_tags, stream_tags, check=True)
        else:
            host = np.asarray(values, dtype=np.float64)
            if host.ndim != 2:
                raise ValueError("feature values must be a 2-d matrix")
            self._set(None, host.shape[1], host, step_tags, stream_tags, check=True)

    @classmethod
    def _from_block(cls, blk: torch.Tensor, d: int, step_tags, stream_tags, check: bool = True,
                    proven_finite: bool = False):
        """Wrap a device block. proven_finite: the caller knows every value is
        finite (e.g. from finite sums of squares of its parts), so the check is
        skipped but recorded as done."""
        fm = cls.__new__(cls)
        fm._set(blk, d, None, step_tags, stream_tags, check and not proven_finite)
        if proven_finite:
            fm._finite_checked = True
        return fm

    def _set(self, blk, d, host, step_tags, stream_tags, check):
        steps = np.asarray(step_tags, dtype=np.int64)
        streams = np.asarray(stream_tags, dtype=np.int64)
        if steps.shape != (d,) or streams.shape != (d,):
            raise ValueError("provenance tags must have one entry per column")
        if check:
            finite = np.all(np.isfinite(host)) if host is not None else block_nonfinite(blk) == 0
            if not finite:
                raise ValueError("feature values must be finite")
        self._blk, self._d, self._host = blk, int(d), host
        self._finite_checked = bool(check)  # values validated finite at construction
        self.step_tags, self.stream_tags = steps, streams

    @classmethod
    def tagged(cls, values, step: int) -> "FeatureMatrix":
        """Wrap a freshly filtered block: all columns from `step`, streams 0..d-1."""
        d = values.shape[1]
        return cls(values, np.full(d, step, dtype=np.int64), np.arange(d, dtype=np.int64))

    @property
    def values(self) -> np.ndarray:
        if self._host is None:
            self._host = download_block(self._blk, self._d)
        return self._host

    def device_block(self) -> torch.Tensor:
        """Padded (n, ld) float64 block on the GPU (uploaded on first use)."""
        if self._blk is None:
            self._blk = upload_block(self._host)
        return self._blk

    @property
    def n(self) -> int:
        return self._blk.shape[0] if self._blk is not None else self._host.shape[0]

    @property
    def d(self) -> int:
        return self._d

    def take(self, cols) -> "FeatureMatrix":
        """Column subset, tags carried along."""
        cols = np.asarray(cols, dtype=np.int64)
        if cols.size and (cols.min() < -self._d or cols.max() >= self._d):
            raise IndexError("column index out of range")
        cols = np.where(cols < 0, cols + self._d, cols)
        src = self.device_block()
        out = torch.zeros((self.n, row_stride(cols.size)), dtype=torch.float64, device=src.device)
        gather_columns(src, cols, out)
        return FeatureMatrix._from_block(out, cols.size, self.step_tags[cols], self.stream_tags[cols],
                                         check=False)

    def with_step(self, step: int) -> "FeatureMatrix":
        fm = FeatureMatrix.__new__(FeatureMatrix)
        fm._set(self._blk, self._d, self._host, np.full(self._d, step, dtype=np.int64), self.stream_tags,
                check=False)
        return fm
