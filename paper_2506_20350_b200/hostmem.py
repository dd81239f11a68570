"""Page-locked host tensors for the host-in / host-out operator calls.

The reference is numpy in / numpy out (``toeplitz.py:287-303``); on the GPU that means a PCIe
copy each way per call.  A host vector held in ``pinned_empty`` / ``pin`` memory goes through
``toep_matvec_host`` (one library call: copy in, apply, copy out, synchronise) and the result
comes back in the same kind of memory.  The blocks come from ``toep_host_alloc`` (cudaHostAlloc):
the copy engines read them at the PCIe rate (1.84 MB in 37 us on the B200 boxes) where torch's
caching host allocator's blocks measured 17-19 GB/s host->device (``tools/hostbuf_probe.py``).

Freed tensors return their block to a small size-keyed cache (cudaHostAlloc costs far more than
a matvec), capped at ``TOEP_HOST_CACHE_MB`` (default 1024) MB of idle blocks.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np
import torch

from . import _lib

_ALIGN = 4096
_CACHE_CAP = int(os.environ.get("TOEP_HOST_CACHE_MB", "1024")) << 20
_cache: dict[int, list[int]] = {}
_live: dict[int, int] = {}  # start address -> bytes of every block handed out and not yet released
_cached_bytes = 0
_mu = threading.Lock()
_types: dict[int, type] = {}


def _release(addr: int, nbytes: int) -> None:
    global _cached_bytes
    with _mu:
        _live.pop(addr, None)
        if _cached_bytes + nbytes <= _CACHE_CAP:
            _cache.setdefault(nbytes, []).append(addr)
            _cached_bytes += nbytes
            return
    _lib.lib().toep_host_free(ctypes.c_void_p(addr))


def _block_type(nbytes: int) -> type:
    t = _types.get(nbytes)
    if t is None:
        def __del__(self, _n=nbytes):
            try:
                _release(ctypes.addressof(self), _n)
            except Exception:  # noqa: BLE001 - interpreter shutdown
                pass
        t = type(f"HostBlock{nbytes}", (ctypes.c_char * nbytes,), {"__del__": __del__})
        _types[nbytes] = t
    return t


def _acquire(nbytes: int) -> int:
    global _cached_bytes
    with _mu:
        free = _cache.get(nbytes)
        if free:
            _cached_bytes -= nbytes
            addr = free.pop()
            _live[addr] = nbytes
            return addr
    out = ctypes.c_void_p()
    _lib.check(_lib.lib().toep_host_alloc(ctypes.c_uint64(nbytes), ctypes.byref(out)), "pinned_empty")
    with _mu:
        _live[int(out.value)] = nbytes
    return int(out.value)


_layouts: dict = {}


def _layout(shape, dtype):
    key = (shape, dtype)
    lay = _layouts.get(key)
    if lay is None:
        shp = (int(shape),) if isinstance(shape, (int, np.integer)) else tuple(int(s) for s in shape)
        count = int(np.prod(shp, dtype=np.int64)) if shp else 1
        nbytes = max(_ALIGN, -(-count * torch.empty((), dtype=dtype).element_size() // _ALIGN) * _ALIGN)
        lay = (shp, count, nbytes, _block_type(nbytes))
        if len(_layouts) < 4096:
            _layouts[key] = lay
    return lay


def pinned_empty(shape, dtype=torch.complex128) -> torch.Tensor:
    """Uninitialised page-locked CPU tensor (``is_pinned()`` is True) from the library allocator."""
    _lib.require_cuda()
    try:
        shp, count, nbytes, btype = _layout(shape, dtype)
    except TypeError:  # unhashable shape (e.g. a list)
        shp, count, nbytes, btype = _layout(tuple(shape), dtype)
    if count == 0:  # torch.frombuffer rejects count=0; an empty pinned tensor needs no block
        return torch.empty(shp, dtype=dtype, pin_memory=True)
    block = btype.from_address(_acquire(nbytes))
    return torch.frombuffer(block, dtype=dtype, count=count).view(shp)


def pin(x, dtype=None) -> torch.Tensor:
    """Copy a numpy array / tensor into a fresh ``pinned_empty`` tensor (complex128 by default)."""
    t = torch.as_tensor(x)
    if t.is_conj():
        t = t.resolve_conj()
    if t.is_neg():
        t = t.resolve_neg()
    out = pinned_empty(t.shape, dtype or (t.dtype if t.is_complex() else torch.complex128))
    out.copy_(t)
    return out


def pinned_view(a: np.ndarray):
    """Tensor view of a C-contiguous numpy array that starts a live library page-locked block (e.g.
    the numpy result of a previous host-path call), else None."""
    if not a.flags.c_contiguous or not a.flags.writeable or a.dtype not in (np.complex128, np.complex64):
        return None
    addr = a.__array_interface__["data"][0]
    with _mu:
        nbytes = _live.get(addr)
    if nbytes is None or a.nbytes > nbytes:
        return None
    return torch.from_numpy(a)


def is_library_block(t: torch.Tensor) -> bool:
    """True when CPU tensor ``t`` starts a live library page-locked block (an O(1) registry lookup;
    torch's ``is_pinned`` asks the driver, microseconds per call on the host path)."""
    return t.data_ptr() in _live
