"""Two-level block-Toeplitz generators and the device MLFFT matvec.

Drop-in for ``toepsolve.toeplitz`` (``/root/reference/pkg/src/toepsolve/toeplitz.py``).
Generators stay host-side numpy structures, exactly as in the reference
(``BlockGenerator1L/2L``, ``embed_1l/2l``, circulant storage order
``[0, 1, .., n-1, -(n-1), .., -1]``).  ``precompute_spectral`` uploads the
generator once and transforms it on the B200; the resulting
``SpectralOperator`` keeps one n0 x n0 block per frequency bin resident in HBM
and every ``matvec`` runs four shared-memory FFT passes and one streaming
per-bin product through ``libtoepcuda``.

Embedding: the reference embeds into a (2n-1)-circulant per level; here each
level uses the smallest 7-smooth length >= 2n-1 (2n at the BASELINE sizes:
60 for n = 30, 128 for n = 64), which represents the same Toeplitz matrix.
``diag_blocks`` therefore has ``l2*l1`` bins instead of ``(2n2-1)(2n1-1)``;
matvec outputs agree with the reference to rounding (asserted in tests).
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass
from typing import Mapping

import numpy as np
import torch

from . import _lib
from ._tensor import restore, to_columns
from . import hostmem as _hostmem
from .hostmem import pin, pinned_empty, pinned_view  # noqa: F401 - public: host vectors for the host-in/out calls
from .errors import BlockShapeMismatch, MissingOffset, ShapeError

__all__ = [
    "BlockGenerator1L",
    "BlockGenerator2L",
    "SpectralOperator",
    "PaddedVector",
    "circulant_offsets",
    "embed_1l",
    "embed_2l",
    "block_fft_1l",
    "block_fft_2l",
    "precompute_spectral",
    "precompute_spectral_stacked",
    "pad_rhs",
    "extract_result",
    "matvec",
    "matvec_transpose",
    "assemble_dense_1l",
    "assemble_dense",
    "generator_from_stacked",
]

PaddedVector = np.ndarray


def circulant_offsets(n: int) -> np.ndarray:
    """Signed offsets in circulant storage order (toeplitz.py:59-61)."""
    return np.concatenate([np.arange(n), np.arange(-(n - 1), 0)])


@dataclass(frozen=True)
class BlockGenerator1L:
    """Level-1 generator: ``column[o % (2n1-1)]`` is the block of offset o (toeplitz.py:64-89)."""

    n1: int
    n0: int
    column: np.ndarray

    def __post_init__(self):
        want = (2 * self.n1 - 1, self.n0, self.n0)
        if self.column.shape != want:
            raise BlockShapeMismatch(f"column shape {self.column.shape} != {want}")

    def block(self, offset: int) -> np.ndarray:
        if abs(offset) >= self.n1:
            raise MissingOffset(f"offset {offset} outside +-{self.n1 - 1}")
        return self.column[offset % (2 * self.n1 - 1)]

    @property
    def stored_scalars(self) -> int:
        return (2 * self.n1 - 1) * self.n0 * self.n0


@dataclass(frozen=True)
class BlockGenerator2L:
    """Level-2 generator: one level-1 generator per level-2 offset (toeplitz.py:92-132)."""

    n2: int
    n1: int
    n0: int
    columns: tuple

    def __post_init__(self):
        if len(self.columns) != 2 * self.n2 - 1:
            raise BlockShapeMismatch(f"expected {2 * self.n2 - 1} level-1 generators, got {len(self.columns)}")
        if any((c.n1, c.n0) != (self.n1, self.n0) for c in self.columns):
            raise BlockShapeMismatch("level-1 generators disagree on (n1, n0)")

    def column(self, offset: int) -> BlockGenerator1L:
        if abs(offset) >= self.n2:
            raise MissingOffset(f"offset {offset} outside +-{self.n2 - 1}")
        return self.columns[offset % (2 * self.n2 - 1)]

    def block(self, offset2: int, offset1: int) -> np.ndarray:
        return self.column(offset2).block(offset1)

    @property
    def dim(self) -> int:
        return self.n2 * self.n1 * self.n0

    @property
    def stored_scalars(self) -> int:
        return (2 * self.n2 - 1) * (2 * self.n1 - 1) * self.n0 * self.n0

    def stacked4(self) -> np.ndarray:
        """(2n2-1, 2n1-1, n0, n0) array in circulant order (no copy when built from one)."""
        base = _STACKED.get(id(self))
        if base is not None and base[0]() is self:
            return base[1]
        return np.stack([c.column for c in self.columns])


# generators built by generator_from_stacked keep their contiguous stacked4 buffer
_STACKED: dict = {}


def generator_from_stacked(stacked4: np.ndarray) -> BlockGenerator2L:
    """Wrap a circulant-ordered (2n2-1, 2n1-1, n0, n0) array as a generator without copying."""
    arr = np.ascontiguousarray(stacked4, dtype=np.complex128)
    if arr.ndim != 4 or arr.shape[2] != arr.shape[3] or arr.shape[0] % 2 == 0 or arr.shape[1] % 2 == 0:
        raise BlockShapeMismatch(f"stacked generator has shape {arr.shape}")
    n2, n1, n0 = (arr.shape[0] + 1) // 2, (arr.shape[1] + 1) // 2, arr.shape[2]
    gen = BlockGenerator2L(n2, n1, n0, tuple(BlockGenerator1L(n1, n0, arr[i]) for i in range(arr.shape[0])))
    key = id(gen)
    _STACKED[key] = (weakref.ref(gen, lambda _r, k=key: _STACKED.pop(k, None)), arr)
    return gen


def embed_1l(blocks: Mapping[int, np.ndarray], n1: int, n0: int) -> BlockGenerator1L:
    """Offsets -(n1-1)..(n1-1) -> circulant-ordered column (toeplitz.py:168-190)."""
    if n1 < 1 or n0 < 1:
        raise ShapeError("n1 and n0 must be positive")
    want = set(range(-(n1 - 1), n1))
    have = set(blocks)
    if have != want:
        raise MissingOffset(f"offset set mismatch: missing {sorted(want - have)}, stray {sorted(have - want)}")
    column = np.empty((2 * n1 - 1, n0, n0), dtype=np.complex128)
    for off, blk in blocks.items():
        a = np.asarray(blk, dtype=np.complex128)
        if a.shape != (n0, n0):
            raise BlockShapeMismatch(f"block at offset {off} has shape {a.shape}, want {(n0, n0)}")
        column[off % (2 * n1 - 1)] = a
    return BlockGenerator1L(n1, n0, column)


def embed_2l(blocks: Mapping[tuple, np.ndarray], n2: int, n1: int, n0: int) -> BlockGenerator2L:
    """(offset2, offset1) -> block map to a two-level generator (toeplitz.py:193-204)."""
    offs2 = circulant_offsets(n2).tolist()
    stray = {o2 for o2, _ in blocks} - set(offs2)
    cols = []
    for o2 in offs2:
        cols.append(embed_1l({o1: b for (p, o1), b in blocks.items() if p == o2}, n1, n0))
    if stray:
        raise MissingOffset(f"stray level-2 offsets {sorted(stray)}")
    return BlockGenerator2L(n2, n1, n0, tuple(cols))


# ---------------------------------------------------------------- operator
class SpectralOperator:
    """Resident transformed generator (toeplitz.py:135-155), owned by libtoepcuda.

    ``diag_blocks`` (a CUDA tensor, ``(l2*l1, n0, n0)``) materialises the
    blocks on demand; the operator itself stores them transposed for the
    streaming product.  Immutable; safe to share between streams.
    """

    def __init__(self, handle: int, info: _lib.OpInfo, device: torch.device):
        self._handle = ctypes.c_void_p(handle)
        self.n2, self.n1, self.n0 = int(info.n2), int(info.n1), int(info.n0)
        self.l2, self.l1 = int(info.l2), int(info.l1)
        self.dtype = torch.complex64 if info.dtype == _lib.TOEP_C64 else torch.complex128
        self.bins = int(info.bins)
        self.resident_bytes = int(info.resident_bytes)
        self.device = device
        self._finalizer = weakref.finalize(self, _destroy, handle)

    @property
    def handle(self):
        return self._handle

    @property
    def dim(self) -> int:
        return self.n2 * self.n1 * self.n0

    @property
    def stored_scalars(self) -> int:
        return self.bins * self.n0 * self.n0

    @property
    def ctype(self) -> int:
        return _lib.TOEP_C64 if self.dtype == torch.complex64 else _lib.TOEP_C128

    @property
    def diag_blocks(self) -> torch.Tensor:
        out = torch.empty((self.bins, self.n0, self.n0), dtype=self.dtype, device=self.device)
        _lib.check(_lib.lib().toep_op_diag_blocks(self._handle, out.data_ptr(), _lib.stream_handle()), "diag_blocks")
        return out

    def fold_left(self, m) -> "SpectralOperator":
        """Operator with blocks ``m @ D_k`` (m: n0 x n0), e.g. the folded P_K^-1 A."""
        mt = torch.as_tensor(np.asarray(m) if not isinstance(m, torch.Tensor) else m)
        mt = mt.to(device=self.device, dtype=torch.complex128).contiguous()
        if tuple(mt.shape) != (self.n0, self.n0):
            raise ShapeError(f"fold matrix shape {tuple(mt.shape)} != {(self.n0, self.n0)}")
        out = ctypes.c_void_p()
        _lib.check(_lib.lib().toep_op_fold_left(self._handle, mt.data_ptr(), _lib.stream_handle(), ctypes.byref(out)),
                   "fold_left")
        return _wrap(out.value, self.device)

    def spectral_apply(self, hat_in: torch.Tensor, hat_out: torch.Tensor, transpose: bool = False) -> None:
        """hat_out[k] = D_k @ hat_in[k] on (bins, n0, w) device tensors (toeplitz.py:300)."""
        w = hat_in.numel() // (self.bins * self.n0)
        _lib.check(_lib.lib().toep_op_spectral_apply(self._handle, hat_in.data_ptr(), hat_out.data_ptr(), w,
                                                     _lib.TOEP_MV_TRANSPOSE if transpose else 0,
                                                     _lib.stream_handle()), "spectral_apply")

    def __repr__(self):
        return (f"SpectralOperator(n2={self.n2}, n1={self.n1}, n0={self.n0}, grid=({self.l2},{self.l1}), "
                f"dtype={self.dtype}, resident={self.resident_bytes / 1e6:.1f} MB)")


def _destroy(handle):
    try:
        _lib.lib().toep_op_destroy(ctypes.c_void_p(handle))
    except Exception:  # interpreter shutdown
        pass


def _wrap(handle: int, device) -> SpectralOperator:
    info = _lib.OpInfo()
    _lib.check(_lib.lib().toep_op_info(ctypes.c_void_p(handle), ctypes.byref(info)), "op_info")
    return SpectralOperator(handle, info, device)


def _smooth7(m: int) -> int:
    """Smallest 7-smooth length >= m (the default circulant length of each level, as op.cu)."""
    n = max(1, int(m))
    while True:
        r = n
        for p in (2, 3, 5, 7):
            while r % p == 0:
                r //= p
        if r == 1:
            return n
        n += 1


def precompute_spectral(gen: BlockGenerator2L, dtype=torch.complex128, embedding=None) -> SpectralOperator:
    """Transform the generator into resident spectral blocks (toeplitz.py:248-253).

    ``dtype``: torch.complex128 (default) or torch.complex64 (the cfg4 c64
    variant; the transform itself runs in complex128 and the blocks are
    rounded once).  ``embedding``: optional (l2, l1) circulant lengths.
    """
    return precompute_spectral_stacked(gen.stacked4(), dtype=dtype, embedding=embedding)


def precompute_spectral_stacked(stacked4, dtype=torch.complex128, embedding=None, slab=None) -> SpectralOperator:
    """``precompute_spectral`` of a circulant-ordered (2n2-1, 2n1-1, n0, n0) block array: a host
    numpy array, or a complex128 CUDA tensor already resident on the device (no upload).

    ``slab=(kx0, kx1)``: keep only the bins of level-1 frequencies [kx0, kx1) (the kx-slab operator
    of the multi-GPU decomposition, built without ever holding the full operator).
    """
    dev = _lib.require_cuda()
    if isinstance(stacked4, torch.Tensor) and stacked4.is_cuda:
        arr = stacked4.to(dtype=torch.complex128).contiguous()
        ptr, on_dev, shape = arr.data_ptr(), 1, tuple(arr.shape)
    else:
        arr = np.ascontiguousarray(stacked4, dtype=np.complex128)
        ptr, on_dev, shape = arr.ctypes.data, 0, arr.shape
    if len(shape) != 4 or shape[2] != shape[3] or shape[0] % 2 == 0 or shape[1] % 2 == 0:
        raise BlockShapeMismatch(f"stacked generator has shape {shape}")
    n2, n1, n0 = (shape[0] + 1) // 2, (shape[1] + 1) // 2, shape[2]
    l2, l1 = (0, 0) if embedding is None else embedding
    kx0, kx1 = (0, 0) if slab is None else (int(slab[0]), int(slab[1]))
    ct = _lib.TOEP_C64 if dtype in (torch.complex64, "complex64", "c64", np.complex64) else _lib.TOEP_C128
    handle = ctypes.c_void_p()
    _lib.check(_lib.lib().toep_op_create_slab(ptr, on_dev, n2, n1, n0, int(l2), int(l1), ct, kx0, kx1,
                                              _lib.stream_handle(), ctypes.byref(handle)), "precompute_spectral")
    del arr
    return _wrap(handle.value, dev)


def _pinned_ok(op: SpectralOperator, t: torch.Tensor) -> bool:
    if t.is_cuda or t.ndim not in (1, 2) or not (t.dtype == op.dtype or t.dtype == torch.complex128):
        return False
    if not (t.is_contiguous() and not t.is_conj() and not t.is_neg()):
        return False
    return _hostmem.is_library_block(t) or t.is_pinned()


def _apply(op: SpectralOperator, u, flags: int, out=None):
    if isinstance(u, torch.Tensor):
        if _pinned_ok(op, u):
            return _apply_pinned(op, u, flags, out)
    elif isinstance(u, np.ndarray) and u.ndim in (1, 2) and out is None:
        return _apply_numpy(op, u, flags)
    x, origin = to_columns(u, keep_c64=(op.dtype == torch.complex64))
    if x.shape[0] != op.dim:
        raise ShapeError(f"rows {x.shape[0]} != operator dim {op.dim}")
    if op.dtype == torch.complex64 and x.dtype == torch.complex128:
        flags |= _lib.TOEP_MV_IO_C128
    res = torch.empty_like(x)
    _lib.check(_lib.lib().toep_matvec(op.handle, x.data_ptr(), res.data_ptr(), x.shape[1], flags,
                                      _lib.stream_handle()), "matvec")
    res = restore(res, origin)
    if out is not None:
        out.copy_(res)
        return out
    return res


def _apply_pinned(op: SpectralOperator, u: torch.Tensor, flags: int, out=None):
    """Pinned host tensor in -> pinned host tensor out, one library call (copy in, apply, copy out,
    synchronise): no device tensors are created per call.  ``out`` (a pinned tensor of u's shape and
    dtype) receives the result instead of a fresh ``pinned_empty`` block."""
    _lib.require_cuda()
    rows = u.shape[0]
    w = 1 if u.ndim == 1 else u.shape[1]
    if rows != op.dim:
        raise ShapeError(f"rows {rows} != operator dim {op.dim}")
    if op.dtype == torch.complex64 and u.dtype == torch.complex128:
        flags |= _lib.TOEP_MV_IO_C128
    if out is None:
        out = pinned_empty(u.shape, u.dtype)
    elif not (isinstance(out, torch.Tensor) and _pinned_ok(op, out) and out.shape == u.shape
              and out.dtype == u.dtype):
        raise ShapeError("out= must be a contiguous pinned CPU tensor of the input's shape and dtype")
    if w:
        _lib.check(_lib.lib().toep_matvec_host(op.handle, u.data_ptr(), out.data_ptr(), w, flags,
                                               _lib.stream_handle()), "matvec")
    return out


def _apply_numpy(op: SpectralOperator, u: np.ndarray, flags: int):
    """The reference's numpy-in / numpy-out call (toeplitz.py:287-303).  The array is handed to
    ``toep_matvec_host`` as is (``TOEP_MV_STAGE_INPUT``: the library's copy threads stage it into
    page-locked memory in chunks, each chunk's DMA issued as soon as it is staged), and the result is
    returned as a numpy array backed by a library page-locked block (released to the block cache when
    the array dies).  A numpy array that already lives in such a block (a previous result) is
    passed through without staging."""
    want = np.complex64 if (op.dtype == torch.complex64 and u.dtype == np.complex64) else np.complex128
    if u.dtype != want or not u.flags.c_contiguous:
        u = np.ascontiguousarray(u, dtype=want)
    if u.shape[0] != op.dim:
        raise ShapeError(f"rows {u.shape[0]} != operator dim {op.dim}")
    t = pinned_view(u)
    if t is not None:
        return _apply_pinned(op, t, flags).numpy()
    _lib.require_cuda()
    w = 1 if u.ndim == 1 else u.shape[1]
    if op.dtype == torch.complex64 and u.dtype == np.complex128:
        flags |= _lib.TOEP_MV_IO_C128
    out = pinned_empty(u.shape, torch.from_numpy(u[:0]).dtype)
    if w:
        _lib.check(_lib.lib().toep_matvec_host(op.handle, u.__array_interface__["data"][0], out.data_ptr(), w,
                                               flags | _lib.TOEP_MV_STAGE_INPUT, _lib.stream_handle()), "matvec")
    return out.numpy()


def matvec(op: SpectralOperator, u, out=None):
    """pad -> DFT -> per-bin D_k multiply -> inverse DFT -> extract (toeplitz.py:287-303).

    numpy in -> numpy out (the reference's convention), CUDA tensor in -> CUDA tensor out, pinned
    CPU tensor in -> pinned CPU tensor out.  ``out`` (optional extension): a preallocated result of
    the same container, shape and dtype, for steady-state loops without per-call allocations.
    """
    return _apply(op, u, 0, out)


def matvec_transpose(op: SpectralOperator, u, out=None):
    """Plain transpose action (toeplitz.py:306-324)."""
    return _apply(op, u, _lib.TOEP_MV_TRANSPOSE, out)


def block_fft_2l(data, n2: int, n1: int, n0: int, direction: str = "forward"):
    """F_{n2} (x) F_{n1} (x) I_{n0} on each column, on the device (toeplitz.py:229-245)."""
    if direction not in ("forward", "inverse"):
        raise ValueError(f"direction must be 'forward' or 'inverse', got {direction!r}")
    x, origin = to_columns(data)
    if min(n2, n1, n0) < 1 or x.shape[0] != n2 * n1 * n0:
        raise ShapeError(f"rows {x.shape[0]} != n2*n1*n0 = {n2 * n1 * n0}")
    out = torch.empty_like(x)
    _lib.check(_lib.lib().toep_block_dft(x.data_ptr(), out.data_ptr(), n2, n1, n0 * x.shape[1],
                                         int(direction == "inverse"), _lib.TOEP_C128, _lib.stream_handle()),
               "block_fft_2l")
    return restore(out, origin)


def block_fft_1l(data, n0: int, direction: str = "forward"):
    """F_L (x) I_{n0} on each column (toeplitz.py:215-226)."""
    if direction not in ("forward", "inverse"):
        raise ValueError(f"direction must be 'forward' or 'inverse', got {direction!r}")
    x, origin = to_columns(data)
    rows = x.shape[0]
    if n0 < 1 or rows % n0:
        raise ShapeError(f"rows {rows} not divisible by block side {n0}")
    out = torch.empty_like(x)
    _lib.check(_lib.lib().toep_block_dft(x.data_ptr(), out.data_ptr(), 1, rows // n0, n0 * x.shape[1],
                                         int(direction == "inverse"), _lib.TOEP_C128, _lib.stream_handle()),
               "block_fft_1l")
    return restore(out, origin)


def pad_rhs(u, n2: int, n1: int, n0: int):
    """Zero-embed a stacked vector into the (2n2-1, 2n1-1) circulant grid (toeplitz.py:256-269).

    The matvec never materialises this (the first FFT pass reads u directly);
    it is provided for API parity.
    """
    x, origin = to_columns(u)
    if x.shape[0] != n2 * n1 * n0:
        raise ShapeError(f"rows {x.shape[0]} != n2*n1*n0 = {n2 * n1 * n0}")
    w = x.shape[1]
    out = torch.zeros(((2 * n2 - 1) * (2 * n1 - 1) * n0, w), dtype=x.dtype, device=x.device)
    out.view(2 * n2 - 1, 2 * n1 - 1, n0, w)[:n2, :n1] = x.view(n2, n1, n0, w)
    return restore(out, origin)


def extract_result(v, n2: int, n1: int, n0: int):
    """Payload rows of a circulant-length vector (toeplitz.py:272-284)."""
    x, origin = to_columns(v)
    if x.shape[0] != (2 * n2 - 1) * (2 * n1 - 1) * n0:
        raise ShapeError(f"rows {x.shape[0]} != circulant length {(2 * n2 - 1) * (2 * n1 - 1) * n0}")
    w = x.shape[1]
    out = x.view(2 * n2 - 1, 2 * n1 - 1, n0, w)[:n2, :n1].reshape(n2 * n1 * n0, w).contiguous()
    return restore(out, origin)


def assemble_dense_1l(gen: BlockGenerator1L) -> np.ndarray:
    """Dense level-1 block-Toeplitz matrix, host (toeplitz.py:327-331)."""
    idx = (np.arange(gen.n1)[:, None] - np.arange(gen.n1)[None, :]) % (2 * gen.n1 - 1)
    return gen.column[idx].transpose(0, 2, 1, 3).reshape(gen.n1 * gen.n0, gen.n1 * gen.n0)


def assemble_dense(gen: BlockGenerator2L) -> np.ndarray:
    """Dense two-level matrix, host, oracle-sized (toeplitz.py:334-345)."""
    s4 = gen.stacked4()
    i2 = (np.arange(gen.n2)[:, None] - np.arange(gen.n2)[None, :]) % (2 * gen.n2 - 1)
    i1 = (np.arange(gen.n1)[:, None] - np.arange(gen.n1)[None, :]) % (2 * gen.n1 - 1)
    full = s4[i2[:, :, None, None], i1[None, None, :, :]]
    return full.transpose(0, 2, 4, 1, 3, 5).reshape(gen.dim, gen.dim)
