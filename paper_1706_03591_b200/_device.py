"""Device plumbing: CUDA availability, streams, padded row-major blocks.

Dense blocks live on the GPU as (n, ld) row-major tensors whose row stride is
a multiple of 32 bytes (one L2 sector), padding columns zero. The padding
never changes a result: zero columns stay zero under the recurrence and add
nothing to any norm or distance.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native

_checked = False


def require_cuda() -> torch.device:
    """The product path has no CPU fallback: fail loudly without a GPU."""
    global _checked
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1706_03591_b200 needs a CUDA device (B200, sm_100a); "
                           "no CPU fallback exists")
    if not _checked:
        _native.load()
        _checked = True
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def row_stride(d: int, dtype: torch.dtype = torch.float64) -> int:
    """Elements per padded row: d rounded up to a 32-byte multiple."""
    per = 32 // torch.empty((), dtype=dtype).element_size()
    return ((d + per - 1) // per) * per


def dtype_code(dtype: torch.dtype) -> int:
    if dtype == torch.float64:
        return _native.CSC_F64
    if dtype == torch.float32:
        return _native.CSC_F32
    raise ValueError(f"unsupported dtype {dtype}")


def torch_dtype(precision: str) -> torch.dtype:
    if precision in ("fp64", "float64", None):
        return torch.float64
    if precision in ("fp32", "float32"):
        return torch.float32
    raise ValueError(f"unknown precision {precision!r}")


def upload_block(x: np.ndarray, dtype: torch.dtype = torch.float64, ld: int | None = None):
    """numpy (n, d) -> padded device block (n, ld) via pinned memory."""
    dev = require_cuda()
    x = np.asarray(x)
    n, d = x.shape
    ld = ld or row_stride(d, dtype)
    host = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    pinned = host.is_pinned()
    if d == ld and dtype == torch.float64:
        return host.to(dev, non_blocking=pinned)
    staged = host.to(dev, non_blocking=pinned)
    out = torch.zeros((n, ld), dtype=dtype, device=dev)
    if n:
        out[:, :d].copy_(staged)
    return out


def download_block(t: torch.Tensor, d: int) -> np.ndarray:
    """Padded device block -> C-contiguous float64 numpy (n, d)."""
    v = t[:, :d]
    if v.dtype != torch.float64:
        v = v.to(torch.float64)
    if not v.is_contiguous():
        v = v.contiguous()
    host = torch.empty(v.shape, dtype=torch.float64, pin_memory=True)
    host.copy_(v, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return host.numpy()


def as_device_block(x, dtype: torch.dtype = torch.float64):
    """Accept numpy or torch (n, d); return (padded block, d, was_numpy)."""
    if isinstance(x, torch.Tensor):
        if x.ndim != 2:
            raise ValueError("signals must be a 2-d matrix")
        n, d = x.shape
        ld = row_stride(d, dtype)
        if x.is_cuda and x.dtype == dtype and x.stride() == (ld, 1) and x.shape[1] == ld:
            return x, d, False
        blk = torch.zeros((n, ld), dtype=dtype, device=require_cuda())
        blk[:, :d].copy_(x)
        return blk, d, False
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 2:
        raise ValueError("signals must be a 2-d matrix")
    return upload_block(x, dtype), x.shape[1], True
