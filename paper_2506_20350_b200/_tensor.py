"""Host <-> device plumbing for the drop-in API.

The reference API is numpy in / numpy out, coercing to complex128
(toeplitz.py:158-165 ``_as_columns``).  Here every call moves its operand to
the CUDA device as a contiguous (rows, w) column block, runs the device path,
and hands the result back in the caller's container: numpy in -> numpy out,
CUDA tensor in -> CUDA tensor out (no copies), pinned CPU tensor in -> pinned
CPU tensor out (asynchronous copies on the current stream).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ShapeError


@dataclass
class Origin:
    kind: str          # "numpy" | "cuda" | "cpu"
    vector: bool
    pinned: bool = False


def to_columns(data, dtype: torch.dtype = torch.complex128, keep_c64: bool = False):
    """Return (device (rows, w) contiguous tensor, Origin)."""
    dev = _lib.require_cuda()
    if isinstance(data, torch.Tensor):
        t = data
        kind = "cuda" if t.is_cuda else "cpu"
        pinned = (not t.is_cuda) and t.is_pinned()
        want = torch.complex64 if (keep_c64 and t.dtype == torch.complex64) else dtype
        t = t.to(device=dev, dtype=want, non_blocking=pinned).resolve_conj().resolve_neg()  # lazy views -> memory
    else:
        arr = np.asarray(data, dtype=np.complex128)
        kind, pinned = "numpy", False
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
        if dtype != torch.complex128:
            t = t.to(dtype)
    if t.ndim == 1:
        return t.reshape(-1, 1).contiguous(), Origin(kind, True, pinned)
    if t.ndim != 2:
        raise ShapeError(f"expected a vector or column block, got ndim={t.ndim}")
    return t.contiguous(), Origin(kind, False, pinned)


def restore(t: torch.Tensor, origin: Origin, out_dtype=None):
    """Device (rows, w) result -> the caller's container and rank."""
    if origin.vector:
        t = t[:, 0]
    if origin.kind == "cuda":
        return t
    if origin.kind == "cpu":
        host = torch.empty(t.shape, dtype=t.dtype, pin_memory=origin.pinned)
        host.copy_(t, non_blocking=origin.pinned)
        if origin.pinned:
            torch.cuda.current_stream().synchronize()
        return host
    out = t.cpu().numpy()
    if out_dtype is not None:
        out = out.astype(out_dtype, copy=False)
    return out


def as_numpy(data) -> np.ndarray:
    if isinstance(data, torch.Tensor):
        return data.detach().cpu().numpy()
    return np.asarray(data)
