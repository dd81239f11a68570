"""Block-diagonal left preconditioners (drop-in for solvers/precond.py of the reference).

P_K = diag(R_00, ..., R_00[, Z_C]) and P_Z = diag(row self block, ...[, Z_C]).
The factorisation of the diagonal block happens once at build time
(precond.py:124-142); applying P^-1 is a device block product with the
precomputed inverse (``toep_block_apply``), batched over every segment and
column, instead of the reference's LAPACK back substitution (precond.py:65-71).
For the solver fast path the element preconditioner is folded into the
spectral operator (``SpectralOperator.fold_left``), so an Arnoldi step pays no
extra HBM traffic for it.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .. import _lib, numerics
from .._tensor import restore, to_columns
from ..errors import ShapeError
from ..toeplitz import assemble_dense_1l

__all__ = [
    "Preconditioner",
    "DenseLUPreconditioner",
    "build_pk",
    "build_pz",
    "identity_preconditioner",
    "apply_precond",
]


@dataclass(frozen=True)
class Preconditioner:
    """Shared-LU block-diagonal preconditioner over array segments + border (precond.py:35-96)."""

    kind: str
    element_lu: numerics.LUFactors | None
    border_lu: numerics.LUFactors | None
    array_dim: int
    nb: int
    _dev: dict = field(default_factory=dict, compare=False, repr=False)

    def __post_init__(self):
        if self.kind not in ("pk", "pz", "none"):
            raise ValueError(f"unknown preconditioner kind {self.kind!r}")
        if self.kind != "none" and self.array_dim % self.element_lu.side:
            raise ShapeError(f"array dim {self.array_dim} not divisible by block side {self.element_lu.side}")

    @property
    def dim(self) -> int:
        return self.array_dim + self.nb

    @property
    def side(self) -> int:
        return self.element_lu.side if self.element_lu is not None else 0

    @property
    def stored_bytes(self) -> int:
        if self.kind == "none":
            return 0
        n = self.element_lu.side ** 2 + (self.border_lu.side ** 2 if self.border_lu else 0)
        return n * 16

    def device_blocks(self):
        """(P^-1 block, P block, border inverse) as device complex128 tensors."""
        if "pinv" not in self._dev:
            dev = _lib.require_cuda()
            lu = self.element_lu
            inv = numerics.block_inverse(lu)
            self._dev["pinv"] = torch.from_numpy(np.ascontiguousarray(inv)).to(dev)
            self._dev["pmat"] = torch.from_numpy(_reassemble(lu)).to(dev)
            self._dev["pinv_h"] = torch.conj_physical(self._dev["pinv"]).T.contiguous()
            if self.border_lu is not None:
                binv = numerics.block_inverse(self.border_lu)
                self._dev["binv"] = torch.from_numpy(binv).to(dev)
                self._dev["binv_h"] = torch.conj_physical(self._dev["binv"]).T.contiguous()
        return self._dev

    def _apply(self, v, adjoint: bool):
        x, origin = to_columns(v)
        if x.shape[0] != self.dim:
            raise ShapeError(f"input shape {tuple(np.shape(v))} incompatible with dim {self.dim}")
        if self.kind == "none":
            return restore(x, origin)
        d = self.device_blocks()
        m = d["pinv_h" if adjoint else "pinv"]
        side = self.element_lu.side
        out = torch.empty_like(x)
        top = x[: self.array_dim].contiguous()
        top_out = out[: self.array_dim]
        _lib.check(_lib.lib().toep_block_apply(m.data_ptr(), side, top.data_ptr(), top_out.data_ptr(),
                                               self.array_dim // side, x.shape[1], _lib.TOEP_C128,
                                               _lib.stream_handle()), "precond apply")
        if self.nb:
            out[self.array_dim:] = d["binv_h" if adjoint else "binv"] @ x[self.array_dim:]
        return restore(out, origin)

    def apply(self, v):
        """P^-1 v (precond.py:90-92)."""
        return self._apply(v, False)

    def apply_adjoint(self, v):
        """P^-H v (precond.py:94-96)."""
        return self._apply(v, True)


def _reassemble(f: numerics.LUFactors) -> np.ndarray:
    """The factored block A from LAPACK-style (lu, ipiv): A[perm[i]] = (L U)[i]."""
    n = f.side
    lu = (np.tril(f.lu, -1) + np.eye(n)) @ np.triu(f.lu)
    perm = np.arange(n)
    for i, p in enumerate(f.piv):
        perm[i], perm[p] = perm[p], perm[i]
    out = np.empty_like(lu)
    out[perm] = lu
    return np.ascontiguousarray(out)


@dataclass(frozen=True)
class DenseLUPreconditioner:
    """Full-matrix LU preconditioner (reference/diagnostic only, precond.py:99-117)."""

    lu: numerics.LUFactors

    @property
    def kind(self) -> str:
        return "dense"

    @property
    def stored_bytes(self) -> int:
        return self.lu.side ** 2 * 16

    def apply(self, v):
        x, origin = to_columns(v)
        inv = torch.from_numpy(numerics.block_inverse(self.lu)).to(x.device)
        return restore(inv @ x, origin)

    def apply_adjoint(self, v):
        x, origin = to_columns(v)
        inv = torch.from_numpy(numerics.block_inverse(self.lu)).to(x.device)
        return restore(inv.conj().T @ x, origin)


def _border_lu(sys):
    return numerics.lu_factor(sys.zc) if sys.nb else None


def build_pk(sys) -> Preconditioner:
    """One shared LU of the element self block R_00 (precond.py:124-131)."""
    return Preconditioner("pk", numerics.lu_factor(sys.gen.block(0, 0)), _border_lu(sys), sys.array_dim, sys.nb)


def build_pz(sys) -> Preconditioner:
    """LU of the assembled row self interaction, side nx*ne (precond.py:134-142)."""
    row = assemble_dense_1l(sys.gen.column(0))
    return Preconditioner("pz", numerics.lu_factor(row), _border_lu(sys), sys.array_dim, sys.nb)


def identity_preconditioner(dim: int) -> Preconditioner:
    return Preconditioner("none", None, None, dim, 0)


def apply_precond(p, v):
    """P^-1 v for a preconditioner object, or v itself for None (precond.py:150-154)."""
    if p is None:
        x, origin = to_columns(v)
        return restore(x, origin)
    return p.apply(v)
