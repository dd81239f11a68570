"""Multi-GPU execution of the hot path: one process per GPU, torch.distributed (NCCL on B200).

The reference has no parallelism.  Work is split only where it
shards:

* ``solve_columns_sharded`` — multi-RHS solves (cfg3): right-hand-side columns are
  independent units, so each rank solves a contiguous column range with the batched
  per-column GMRES and nothing crosses ranks in the data path; X and the per-column
  reports are gathered once at the end.
* ``SlabOperator`` — one large array (cfg4): the Krylov vectors are distributed by array
  rows, the spectral blocks by level-1 frequency slab.  A matvec is: local level-1 DFT of
  the rank's rows -> all-to-all (rows -> kx slabs) -> local level-2 DFT, per-bin product
  and inverse level-2 DFT on the slab -> all-to-all back -> local inverse level-1 DFT.
  Only the Ny kept rows are exchanged (16.8 MB per transpose).
* single-RHS cfg2 does not shard usefully: ``bench.py --gpus N`` runs replicas.

The local stages go through libtoepcuda (``toep_matvec_stage``); tests inject CPU stage
doubles to exercise the decomposition / exchange logic on gloo with world size 2.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .errors import NoConvergence, ShapeError

__all__ = ["column_range", "row_range", "solve_columns_sharded", "SlabOperator", "slab_ranges"]


def column_range(w: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous split of w columns (first w % world ranks get one more)."""
    per, rem = divmod(w, world)
    c0 = rank * per + min(rank, rem)
    return c0, c0 + per + (1 if rank < rem else 0)


row_range = column_range
slab_ranges = column_range


def _gather_cols(x_local: torch.Tensor, w: int, world: int, group) -> torch.Tensor:
    """All-gather column shards (n, w_r) into (n, w) on every rank."""
    n = x_local.shape[0]
    per = -(-w // world)
    buf = torch.zeros((n, per), dtype=x_local.dtype, device=x_local.device)
    buf[:, : x_local.shape[1]] = x_local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf.contiguous(), group=group)
    cols = []
    for r in range(world):
        c0, c1 = column_range(w, world, r)
        cols.append(parts[r][:, : c1 - c0])
    return torch.cat(cols, dim=1)


def solve_columns_sharded(op, p, rhs, cfg, group=None, solver=None, method: str = "sequential"):
    """Column-sharded ``solve_multi_rhs_sequential`` (gmres.py:304-336) over the process group.

    Every rank passes the full (n, W) right-hand side (or just its own columns via
    ``rhs_is_local``-free convention: the full block is sliced here); each solves its column
    range, then X and the reports are all-gathered, so every rank returns the full result.
    ``solver(op, p, block, cfg, method)`` defaults to the device batched solver.
    """
    if solver is None:
        from .solvers.gmres import solve_multi_rhs_sequential as solver
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    full = torch.as_tensor(rhs) if not isinstance(rhs, torch.Tensor) else rhs
    if full.ndim != 2:
        raise ShapeError(f"rhs must be a column block, got ndim={full.ndim}")
    w = full.shape[1]
    c0, c1 = column_range(w, world, rank)
    local = full[:, c0:c1].contiguous()
    failed_local = False
    try:
        x_local, reports = solver(op, p, local, cfg, method)
    except NoConvergence as exc:
        x_local, reports, failed_local = exc.solution, exc.reports, True
    x_local = torch.as_tensor(x_local)
    if world == 1:
        if failed_local:
            raise NoConvergence("columns did not converge", solution=x_local, reports=reports)
        return x_local, reports
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    x_all = _gather_cols(x_local.to(dev), w, world, group)
    gathered = [None] * world
    dist.all_gather_object(gathered, reports, group=group)
    all_reports = [r for part in gathered for r in part]
    if any(not r.converged for r in all_reports):
        bad = [i for i, r in enumerate(all_reports) if not r.converged]
        raise NoConvergence(f"columns {bad} did not converge within {cfg.max_iter} iterations", solution=x_all,
                            reports=all_reports)
    return x_all, all_reports


class SlabOperator:
    """Row / kx-slab decomposed matvec of one large array over the process group.

    Rank r owns array rows ``row_range(Ny, P, r)`` of every (n, W) vector (layout
    ``(rows, Nx, Nb, W)``) and the spectral blocks of level-1 frequencies
    ``slab_ranges(L1, P, r)``.  ``stages`` provides the three local steps (default: the
    device kernels of libtoepcuda):

    * ``fwd_x(u_rows (ny_r, n1, inner)) -> (ny_r, L1, inner)``
    * ``spectral(x1_slab (n2, kxs, inner)) -> (n2, kxs, inner)`` — level-2 DFT, per-bin product
      with the slab's blocks, inverse level-2 DFT (kept rows)
    * ``inv_x(x2_rows (ny_r, L1, inner)) -> (ny_r, n1, inner)`` with the 1/(L1 L2) scale
    """

    def __init__(self, n2: int, n1: int, n0: int, l2: int, l1: int, stages, group=None):
        self.n2, self.n1, self.n0, self.l2, self.l1 = n2, n1, n0, l2, l1
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.rows = row_range(n2, self.world, self.rank)
        self.slab = slab_ranges(l1, self.world, self.rank)
        self.stages = stages

    @classmethod
    def from_generator(cls, gen, group=None, dtype=torch.complex128):
        """Device slab operator: each rank keeps only its kx slab of the spectral blocks."""
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        st = DeviceSlabStages(gen, world, rank, dtype)
        return cls(gen.n2, gen.n1, gen.n0, st.l2, st.l1, st, group)

    @property
    def local_dim(self) -> int:
        return (self.rows[1] - self.rows[0]) * self.n1 * self.n0

    def _exchange(self, send_blocks, recv_shapes, like):
        """all-to-all of a list of per-destination blocks; returns per-source blocks."""
        if self.world == 1:
            return [send_blocks[0]]
        send = torch.cat([b.reshape(-1) for b in send_blocks]).contiguous()
        out_sizes = [int(np.prod(s)) for s in recv_shapes]
        recv = torch.empty(sum(out_sizes), dtype=like.dtype, device=like.device)
        in_sizes = [b.numel() for b in send_blocks]
        if like.is_complex():
            dist.all_to_all_single(torch.view_as_real(recv), torch.view_as_real(send),
                                   output_split_sizes=out_sizes, input_split_sizes=in_sizes, group=self.group)
        else:
            dist.all_to_all_single(recv, send, output_split_sizes=out_sizes, input_split_sizes=in_sizes,
                                   group=self.group)
        parts, off = [], 0
        for shape, sz in zip(recv_shapes, out_sizes):
            parts.append(recv[off:off + sz].reshape(shape))
            off += sz
        return parts

    def matvec_local(self, u_local: torch.Tensor) -> torch.Tensor:
        """Distributed matvec: this rank's rows in, this rank's rows out ((rows*n1*n0, W))."""
        if u_local.ndim == 1:
            u_local = u_local[:, None]
        w = u_local.shape[1]
        inner = self.n0 * w
        y0, y1 = self.rows
        ny = y1 - y0
        if u_local.shape[0] != ny * self.n1 * self.n0:
            raise ShapeError(f"local rows {u_local.shape[0]} != {ny * self.n1 * self.n0}")
        x1 = self.stages.fwd_x(u_local.reshape(ny, self.n1, inner))            # (ny, L1, inner)
        slabs = [slab_ranges(self.l1, self.world, q) for q in range(self.world)]
        rows = [row_range(self.n2, self.world, q) for q in range(self.world)]
        k0, k1 = self.slab
        send = [x1[:, a:b, :] for (a, b) in slabs]
        recv_shapes = [((r1 - r0), k1 - k0, inner) for (r0, r1) in rows]
        got = self._exchange(send, recv_shapes, x1)
        x1_slab = torch.cat(got, dim=0).contiguous()                           # (n2, kxs, inner)
        x2_slab = self.stages.spectral(x1_slab)                                # (n2, kxs, inner)
        send2 = [x2_slab[r0:r1] for (r0, r1) in rows]
        recv2 = [(ny, b - a, inner) for (a, b) in slabs]
        back = self._exchange(send2, recv2, x2_slab)
        x2 = torch.cat(back, dim=1).contiguous()                               # (ny, L1, inner)
        v = self.stages.inv_x(x2)                                              # (ny, n1, inner)
        return v.reshape(ny * self.n1 * self.n0, w)

    # distributed reductions for a Krylov solver over row-distributed vectors
    def dot(self, a: torch.Tensor, b: torch.Tensor) -> complex:
        t = torch.sum(torch.conj(a) * b).reshape(1)
        if self.world > 1:
            tr = torch.view_as_real(t).contiguous()
            dist.all_reduce(tr, group=self.group)
            t = torch.view_as_complex(tr)
        return complex(t.item())

    def norm(self, a: torch.Tensor) -> float:
        t = torch.sum(a.real * a.real + a.imag * a.imag).reshape(1)
        if self.world > 1:
            dist.all_reduce(t, group=self.group)
        return float(t.sqrt().item())


def gmres_slab(op: SlabOperator, p, b_local, cfg):
    """GMRES (gmres.py:98-249 semantics) on row-distributed vectors of a SlabOperator.

    The device Arnoldi engine (toep_gmres) runs on every rank over the local rows; the
    matvec is the distributed ``op.matvec_local`` (two all-to-alls), every inner product and
    norm is all-reduced over the group on the device stream, so all ranks follow identical
    scalar recurrences (same iterations, same stop step).  ``p``: None or an element-block
    preconditioner (P_K, local to each row block).  Returns this rank's rows of x.
    """
    from .solvers.gmres import _run
    from .errors import NoConvergence
    from ._tensor import to_columns, restore

    b, origin = to_columns(b_local)
    if b.shape[0] != op.local_dim:
        raise ShapeError(f"local rhs rows {b.shape[0]} != {op.local_dim}")
    group = op.group
    world = op.world

    def allreduce(t):
        if world > 1:
            dist.all_reduce(t, group=group)

    x, report = _run(lambda v: op.matvec_local(v), p, b, cfg, prefer_numpy=False, allreduce=allreduce)
    report.method = "gmres-slab"
    xo = restore(x, origin)
    if not report.converged:
        raise NoConvergence(f"distributed GMRES stopped after {report.iterations} iterations", solution=xo,
                            report=report)
    return xo, report


class DeviceSlabStages:
    """The three local stages of SlabOperator on the device (toep_matvec_stage)."""

    def __init__(self, gen, world: int, rank: int, dtype):
        from .toeplitz import precompute_spectral

        self.l2 = self.l1 = None
        full = precompute_spectral(gen, dtype=dtype)
        self.l2, self.l1 = full.l2, full.l1
        k0, k1 = slab_ranges(full.l1, world, rank)
        out = ctypes.c_void_p()
        _lib.check(_lib.lib().toep_op_slab(full.handle, k0, k1, _lib.stream_handle(), ctypes.byref(out)), "op_slab")
        from .toeplitz import _wrap

        self.op = _wrap(out.value, full.device)
        del full
        self.k0, self.k1 = k0, k1
        self.n2, self.n1, self.n0 = gen.n2, gen.n1, gen.n0

    def _stage(self, stage: int, x: torch.Tensor, out_shape, count: int):
        x = x.contiguous()
        out = torch.empty(out_shape, dtype=x.dtype, device=x.device)
        w = x.shape[-1] // self.n0
        _lib.check(_lib.lib().toep_matvec_stage(self.op.handle, stage, x.data_ptr(), out.data_ptr(), w, count,
                                                _lib.stream_handle()), f"matvec_stage {stage}")
        return out

    def fwd_x(self, u_rows):
        ny, _, inner = u_rows.shape
        return self._stage(0, u_rows, (ny, self.l1, inner), ny)

    def spectral(self, x1_slab):
        n2, kxs, inner = x1_slab.shape
        return self._stage(1, x1_slab, (n2, kxs, inner), kxs)

    def inv_x(self, x2_rows):
        ny, _, inner = x2_rows.shape
        return self._stage(2, x2_rows, (ny, self.n1, inner), ny)
