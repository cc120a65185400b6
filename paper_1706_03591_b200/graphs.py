"""Graph container and on-device Laplacians (mirror of cscluster.graphs).

Reference: /root/reference/pkg/src/cscluster/graphs.py
  Graph            graphs.py:15-80   (same validation, canonical order, API)
  graphs_equal     graphs.py:83-90
  LaplacianMatrix  graphs.py:326-336 (same fields; CSR lives on the GPU, the
                                      SciPy `matrix` is materialised lazily)
  laplacian        graphs.py:339-362 (built on device by csc_laplacian_build,
                                      bit-identical values and structure)

Extension for time-evolving graphs (north_star (4)): ``Graph.apply_delta``
returns the next graph from sorted delete/insert code lists and keeps the
edge set on the GPU (csc_edge_delta), so a dynamic step rebuilds its CSR
without re-uploading or re-sorting the whole edge list.
"""
from __future__ import annotations

import ctypes

import numpy as np
import scipy.sparse as sp
import torch

from . import _native
from ._device import dtype_code, ptr, require_cuda, stream

LAPLACIAN_VARIANTS = ("combinatorial", "normalized")


class Graph:
    """Immutable undirected weighted graph; each edge stored once with i < j.

    Construction canonicalizes endpoint order, sorts edges by code i*n+j and
    rejects self-loops, duplicates, nonpositive weights and out-of-range
    indices (graphs.py:29-54) — on the GPU (csc_graph_canonicalize: validation
    flags, stable radix sort of the codes, duplicate scan), for every non-empty
    edge list. The graph then holds its edges on the GPU and materialises the
    host arrays only when asked.
    """

    def __init__(self, n: int, edge_i, edge_j, edge_w):
        if n < 0:
            raise ValueError("node count must be nonnegative")
        i = np.asarray(edge_i, dtype=np.int64).ravel()
        j = np.asarray(edge_j, dtype=np.int64).ravel()
        w = np.asarray(edge_w, dtype=np.float64).ravel()
        if not (i.shape == j.shape == w.shape):
            raise ValueError("edge arrays must have equal length")
        if i.size:  # K9 runs on the GPU (no CPU fallback: raises without CUDA)
            self._canonicalize_on_device(int(n), i, j, w)
            return
        self._init(int(n), i, j, w, None, 0)

    def _canonicalize_on_device(self, n, i, j, w):
        """K9 on the GPU: validation flags, stable radix sort of the codes, duplicate check."""
        dev = require_cuda()
        m = i.size
        ti, tj, tw = (torch.from_numpy(a).to(dev) for a in (i, j, w))
        codes = torch.empty(m, dtype=torch.int64, device=dev)
        w_sorted = torch.empty(m, dtype=torch.float64, device=dev)
        flags = np.zeros(4, dtype=np.int32)
        _native.call("csc_graph_canonicalize", n, m, ptr(ti), ptr(tj), ptr(tw), ptr(codes), ptr(w_sorted),
                     flags.ctypes.data, stream())
        for flag, msg in zip(flags, ("edge endpoint out of range [0, n)", "self-loops are not allowed",
                                     "edge weights must be positive",
                                     "duplicate edges (after canonicalizing endpoint order)")):
            if flag:
                raise ValueError(msg)
        self._init(n, None, None, None, codes, m)
        unit = bool(np.all(w == 1.0))
        object.__setattr__(self, "_unit", unit)
        object.__setattr__(self, "_w_dev", None if unit else w_sorted)

    def _init(self, n, i, j, w, codes_dev, m):
        object.__setattr__(self, "n", n)
        object.__setattr__(self, "_i", i)
        object.__setattr__(self, "_j", j)
        object.__setattr__(self, "_w", w)
        object.__setattr__(self, "_codes_dev", codes_dev)
        object.__setattr__(self, "_m", m)
        object.__setattr__(self, "_unit", None)
        object.__setattr__(self, "_dev_edges", None)
        object.__setattr__(self, "_cache", {})

    def __setattr__(self, name, value):
        raise AttributeError("Graph is immutable")

    # -- host view (reference API) -------------------------------------------
    def _host(self):
        if self._i is None:
            codes = self._codes_dev.cpu().numpy()
            object.__setattr__(self, "_i", codes // self.n)
            object.__setattr__(self, "_j", codes % self.n)
            wd = getattr(self, "_w_dev", None)
            object.__setattr__(self, "_w", wd.cpu().numpy() if wd is not None else np.ones(codes.size))
        return self._i, self._j, self._w

    @property
    def edge_i(self) -> np.ndarray:
        return self._host()[0]

    @property
    def edge_j(self) -> np.ndarray:
        return self._host()[1]

    @property
    def edge_w(self) -> np.ndarray:
        return self._host()[2]

    @property
    def m(self) -> int:
        """Number of undirected edges."""
        return self._m

    @property
    def degrees(self) -> np.ndarray:
        """Weighted degree per node (graphs.py:61-66)."""
        if "degrees" not in self._cache:
            i, j, w = self._host()
            deg = np.bincount(i, weights=w, minlength=self.n)
            deg += np.bincount(j, weights=w, minlength=self.n)
            self._cache["degrees"] = deg
        return self._cache["degrees"]

    @property
    def adjacency(self) -> sp.csr_matrix:
        """Symmetric CSR adjacency, both orientations (graphs.py:68-76)."""
        if "adjacency" not in self._cache:
            i, j, w = self._host()
            a = sp.csr_matrix((np.concatenate([w, w]), (np.concatenate([i, j]), np.concatenate([j, i]))),
                              shape=(self.n, self.n))
            a.sort_indices()
            self._cache["adjacency"] = a
        return self._cache["adjacency"]

    def edge_codes(self) -> np.ndarray:
        """Canonical pair code i*n + j per edge (i < j); sorted ascending."""
        if self._codes_dev is not None and self._i is None:
            return self._codes_dev.cpu().numpy()
        i, j, _ = self._host()
        return i * self.n + j

    # -- device view -------------------------------------------------------------
    def unit_weights(self) -> bool:
        if self._unit is None:
            object.__setattr__(self, "_unit", bool(self._w is None or np.all(self._w == 1.0)))
        return self._unit

    def device_codes(self) -> torch.Tensor:
        """Sorted int64 edge codes on the GPU."""
        if self._codes_dev is None:
            dev = require_cuda()
            i, j, _ = self._host()
            codes = torch.from_numpy(i * self.n + j).to(dev, non_blocking=False)
            object.__setattr__(self, "_codes_dev", codes)
        return self._codes_dev

    def device_edges(self):
        """(lo, hi, w-or-None) int64/int64/float64 tensors on the GPU."""
        if self._dev_edges is None:
            dev = require_cuda()
            if self._i is not None:
                lo = torch.from_numpy(self._i).to(dev)
                hi = torch.from_numpy(self._j).to(dev)
            else:
                codes = self._codes_dev
                lo = torch.empty_like(codes)
                hi = torch.empty_like(codes)
                _native.call("csc_codes_split", self.n, ptr(codes), self.m, ptr(lo), ptr(hi), stream())
            wd = getattr(self, "_w_dev", None)
            if self.unit_weights():
                w = None
            elif wd is not None:
                w = wd
            else:
                w = torch.from_numpy(self._host()[2]).to(dev)
            object.__setattr__(self, "_dev_edges", (lo, hi, w))
        return self._dev_edges

    def apply_delta(self, deletes, inserts) -> "Graph":
        """Next graph: remove `deletes`, add `inserts` (canonical codes lo*n+hi).

        Unit-weight graphs only (the perturbation models insert unit edges,
        graphs.py:270-272). Deletions must be edges of this graph and
        insertions must be absent from the result of the deletions. Host lists
        are sorted on the host; device tensors (the device generators' sorted
        lists) are used in place. The merged edge set stays on the GPU.
        """
        if not self.unit_weights():
            raise ValueError("apply_delta supports unit-weight graphs only")
        dev = require_cuda()
        if isinstance(deletes, torch.Tensor) or isinstance(inserts, torch.Tensor):
            # device lists (generators.edge_churn_device / node_switch_device): sorted, unique
            d_t = torch.as_tensor(deletes, dtype=torch.int64, device=dev).contiguous()
            i_t = torch.as_tensor(inserts, dtype=torch.int64, device=dev).contiguous()
            if i_t.numel():
                lo, hi = i_t // self.n, i_t % self.n
                if not bool(((i_t >= 0) & (lo < hi) & (hi < self.n)).all()):
                    raise ValueError("inserted codes must be canonical pairs i*n+j with i < j < n")
            nd, ni = d_t.numel(), i_t.numel()
        else:
            dl = _sorted_codes(deletes)
            il = _sorted_codes(inserts)
            if il.size:
                lo, hi = il // self.n, il % self.n
                if il.min() < 0 or np.any(lo >= hi) or hi.max() >= self.n:
                    raise ValueError("inserted codes must be canonical pairs i*n+j with i < j < n")
            d_t = torch.from_numpy(dl).to(dev)
            i_t = torch.from_numpy(il).to(dev)
            nd, ni = dl.size, il.size
        prev = self.device_codes()
        m_new = self.m - nd + ni
        out = torch.empty(max(m_new, 1), dtype=torch.int64, device=dev)
        got = ctypes.c_int64(0)
        _native.call("csc_edge_delta", self.n, ptr(prev), self.m, ptr(d_t), nd, ptr(i_t), ni,
                     ptr(out), out.numel(), ctypes.byref(got), stream())
        g = Graph.__new__(Graph)
        g._init(self.n, None, None, None, out[:m_new], int(got.value))
        object.__setattr__(g, "_unit", True)
        return g


def _sorted_codes(codes) -> np.ndarray:
    """Sorted unique int64 codes; lists that already are (the generators' and
    set-difference outputs) pass with one O(m) check instead of a sort."""
    c = np.asarray(codes, dtype=np.int64).ravel()
    if c.size > 1 and not np.all(c[1:] > c[:-1]):
        c = np.unique(c)
    return c


def graphs_equal(a: Graph, b: Graph) -> bool:
    return (a.n == b.n and a.m == b.m and np.array_equal(a.edge_i, b.edge_i)
            and np.array_equal(a.edge_j, b.edge_j) and np.array_equal(a.edge_w, b.edge_w))


class _ChebPlan:
    """Owner of a csc_chebop handle (M = I - scale*L in one dtype + schedule)."""

    def __init__(self, handle, n, nnz, n_long, n_seg, dtype):
        self.handle, self.n, self.nnz, self.n_long, self.n_seg, self.dtype = \
            handle, n, nnz, n_long, n_seg, dtype
        b, cv2 = ctypes.c_int32(0), ctypes.c_double(0.0)
        _native.call("csc_chebop_schedule", handle, ctypes.byref(b), ctypes.byref(cv2))
        self.binned, self.len_cv2 = bool(b.value), float(cv2.value)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _native.lib().csc_chebop_destroy(h)
            except Exception:
                pass
            self.handle = None


def export_plan(plan: _ChebPlan):
    """(indptr, indices, vals, long_rows, seg_off) of a plan as numpy arrays."""
    dev = require_cuda()
    ip = torch.empty(plan.n + 1, dtype=torch.int32, device=dev)
    ix = torch.empty(max(plan.nnz, 1), dtype=torch.int32, device=dev)
    vv = torch.empty(max(plan.nnz, 1), dtype=plan.dtype, device=dev)
    lr = torch.empty(max(plan.n_long, 1), dtype=torch.int32, device=dev)
    so = torch.empty(plan.n_long + 1, dtype=torch.int32, device=dev)
    _native.call("csc_chebop_export", plan.handle, ptr(ip), ptr(ix), ptr(vv), ptr(lr), ptr(so), stream())
    return (ip.cpu().numpy(), ix[:plan.nnz].cpu().numpy(), vv[:plan.nnz].cpu().numpy(),
            lr[:plan.n_long].cpu().numpy(), so.cpu().numpy() if plan.n_long else np.zeros(1, np.int32))


class LaplacianMatrix:
    """Sparse symmetric Laplacian plus an upper bound on its top eigenvalue.

    Same fields as graphs.py:326-336. The CSR (int32 indptr/indices, float64
    values, sorted columns) is resident on the GPU; ``matrix`` returns the
    SciPy view, copied to the host on first access. Built from a SciPy matrix,
    the device copy is made on first use.
    """

    def __init__(self, matrix=None, variant: str = "normalized", lambda_max_bound: float = 2.0):
        self._matrix = None if matrix is None else sp.csr_matrix(matrix)
        self.variant = variant
        self.lambda_max_bound = float(lambda_max_bound)
        self._dev = None
        self._n = None if matrix is None else int(self._matrix.shape[0])
        self._plans = {}

    @classmethod
    def _from_device(cls, indptr, indices, data, n, variant, bound):
        lap = cls(None, variant, bound)
        lap._dev = (indptr, indices, data)
        lap._n = int(n)
        return lap

    @property
    def n(self) -> int:
        return self._n

    @property
    def nnz(self) -> int:
        return int(self._dev[1].numel()) if self._dev is not None else int(self._matrix.nnz)

    @property
    def matrix(self) -> sp.csr_matrix:
        if self._matrix is None:
            ip, ix, dv = (t.cpu().numpy() for t in self._dev)
            m = sp.csr_matrix((dv, ix, ip), shape=(self._n, self._n))
            m.has_sorted_indices = True
            self._matrix = m
        return self._matrix

    def device_csr(self):
        """(indptr int32, indices int32, data float64) on the GPU."""
        if self._dev is None:
            dev = require_cuda()
            m = self._matrix
            if not m.has_sorted_indices:
                m = m.sorted_indices()
            self._dev = (torch.from_numpy(m.indptr.astype(np.int32)).to(dev),
                         torch.from_numpy(m.indices.astype(np.int32)).to(dev),
                         torch.from_numpy(m.data.astype(np.float64)).to(dev))
        return self._dev

    def plan(self, scale: float, dtype: torch.dtype = torch.float64) -> _ChebPlan:
        """Cached Chebyshev operator M = I - scale*L for one dtype."""
        key = (float(scale), dtype)
        if key not in self._plans:
            ip, ix, dv = self.device_csr()
            h = ctypes.c_void_p()
            _native.call("csc_chebop_create", ptr(ip), ptr(ix), ptr(dv), self.n, ix.numel(), float(scale),
                         dtype_code(dtype), stream(), ctypes.byref(h))
            info = [ctypes.c_int64() for _ in range(4)]
            _native.call("csc_chebop_info", h, *[ctypes.byref(v) for v in info])
            self._plans[key] = _ChebPlan(h, *(v.value for v in info), dtype)
        return self._plans[key]


def laplacian(g: Graph, variant: str = "normalized") -> LaplacianMatrix:
    """Combinatorial (D - W) or symmetric normalized Laplacian, built on the GPU.

    Bit-identical to graphs.py:339-362: isolated nodes get an empty row in the
    normalized variant; the bound is 2 (normalized) or twice the maximum
    weighted degree (combinatorial, 0 for an edgeless graph).
    """
    if variant not in LAPLACIAN_VARIANTS:
        raise ValueError(f"unknown Laplacian variant {variant!r}")
    dev = require_cuda()
    n, m = g.n, g.m
    lo, hi, w = g.device_edges()
    cap = 2 * m + n
    indptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
    indices = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    data = torch.empty(max(cap, 1), dtype=torch.float64, device=dev)
    nnz = ctypes.c_int64(0)
    bound = ctypes.c_double(0.0)
    code = _native.CSC_LAP_NORMALIZED if variant == "normalized" else _native.CSC_LAP_COMBINATORIAL
    _native.call("csc_laplacian_build", n, m, ptr(lo), ptr(hi), ptr(w), code, ptr(indptr), ptr(indices),
                 ptr(data), cap, None, ctypes.byref(nnz), ctypes.byref(bound), stream())
    k = int(nnz.value)
    return LaplacianMatrix._from_device(indptr, indices[:k], data[:k], n, variant, bound.value)
