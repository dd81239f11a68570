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

Exchange modes of ``SlabOperator``: ``"collective"`` (``all_to_all_single`` through the process
group: NCCL on GPUs, gloo in the CPU tests) and ``"peer"`` (B200 / NVSwitch): the DFT pass that
produces each exchange stores its output rows straight into the owning rank's receive buffer
(CUDA IPC mapping over NVLink) and bumps that rank's arrival counter; the consumer's stream waits
on its counter.  The all-to-all disappears into the DFT's final store (``PeerExchange``).

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

__all__ = ["column_range", "row_range", "solve_columns_sharded", "SlabOperator", "slab_ranges", "PeerExchange",
           "scatter_plan"]


def column_range(w: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous split of w columns (first w % world ranks get one more)."""
    per, rem = divmod(w, world)
    c0 = rank * per + min(rank, rem)
    return c0, c0 + per + (1 if rank < rem else 0)


row_range = column_range
slab_ranges = column_range


def _gather_cols(x_local: torch.Tensor, w: int, world: int, group, root: int | None) -> torch.Tensor | None:
    """Column shards (n, w_r) -> (n, w) on ``root`` (``None``: on every rank); other ranks get None."""
    n = x_local.shape[0]
    per = -(-w // world)
    buf = torch.zeros((n, per), dtype=x_local.dtype, device=x_local.device)
    buf[:, : x_local.shape[1]] = x_local
    rank = dist.get_rank(group)
    rv = torch.view_as_real if buf.is_complex() else (lambda t: t)  # gloo has no complex collectives
    if root is None:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather([rv(t) for t in parts], rv(buf), group=group)
    else:
        parts = [torch.empty_like(buf) for _ in range(world)] if rank == root else None
        dist.gather(rv(buf), [rv(t) for t in parts] if parts is not None else None,
                    dst=dist.get_global_rank(group, root) if group is not None else root, group=group)
        if rank != root:
            return None
    cols = []
    for r in range(world):
        c0, c1 = column_range(w, world, r)
        cols.append(parts[r][:, : c1 - c0])
    return torch.cat(cols, dim=1)


def solve_columns_sharded(op, p, rhs, cfg, group=None, solver=None, method: str = "sequential",
                          gather: str = "root"):
    """Column-sharded ``solve_multi_rhs_sequential`` (gmres.py:304-336) over the process group.

    Every rank passes the full (n, W) right-hand side (the rank's column range is sliced here) and
    solves its columns with no communication in the data path.  ``gather="root"`` (default):
    rank 0 receives X (n, W) and every column's report, the other ranks return their own column
    block and reports; ``gather="all"``: every rank returns the full result.  A column that did not
    converge raises ``NoConvergence`` on every rank (one all-reduced flag).
    ``solver(op, p, block, cfg, method)`` defaults to the device batched solver.
    """
    if gather not in ("root", "all"):
        raise ValueError(f"gather must be 'root' or 'all', got {gather!r}")
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
    try:
        x_local, reports = solver(op, p, local, cfg, method)
    except NoConvergence as exc:
        x_local, reports = exc.solution, exc.reports
    x_local = torch.as_tensor(x_local)
    if world == 1:
        if any(not r.converged for r in reports):
            bad = [i for i, r in enumerate(reports) if not r.converged]
            raise NoConvergence(f"columns {bad} did not converge within {cfg.max_iter} iterations",
                                solution=x_local, reports=reports)
        return x_local, reports
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    root = None if gather == "all" else 0
    x_all = _gather_cols(x_local.to(dev), w, world, group, root)
    if root is None:
        got = [None] * world
        dist.all_gather_object(got, reports, group=group)
    else:
        got = [None] * world if rank == root else None
        dist.gather_object(reports, got, dst=dist.get_global_rank(group, root) if group is not None else root,
                           group=group)
    failed = torch.tensor([sum(1 for r in reports if not r.converged)], dtype=torch.int64, device=dev)
    dist.all_reduce(failed, group=group)
    if got is not None:
        all_reports = [r for part in got for r in part]
        x_out = x_all
    else:
        all_reports, x_out = reports, x_local
    if int(failed.item()):
        bad = [c0 + i for i, r in enumerate(reports) if not r.converged] if got is None else \
            [i for i, r in enumerate(all_reports) if not r.converged]
        raise NoConvergence(f"{int(failed.item())} columns did not converge within {cfg.max_iter} iterations "
                            f"(this rank's view: {bad})", solution=x_out, reports=all_reports)
    return x_out, all_reports


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

    def __init__(self, n2: int, n1: int, n0: int, l2: int, l1: int, stages, group=None,
                 exchange: str = "collective"):
        if exchange not in ("collective", "peer"):
            raise ValueError(f"exchange must be 'collective' or 'peer', got {exchange!r}")
        self.n2, self.n1, self.n0, self.l2, self.l1 = n2, n1, n0, l2, l1
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.rows = row_range(n2, self.world, self.rank)
        self.slab = slab_ranges(l1, self.world, self.rank)
        self.stages = stages
        self.exchange = exchange
        self._peer = {}  # w -> PeerExchange

    @classmethod
    def from_generator(cls, gen, group=None, dtype=torch.complex128, exchange: str = "collective"):
        """Device slab operator: each rank transforms and keeps only its kx slab of the spectral
        blocks.  ``gen``: a generator, or the stacked blocks (host array / CUDA tensor)."""
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        st = DeviceSlabStages(gen, world, rank, dtype)
        return cls(st.n2, st.n1, st.n0, st.l2, st.l1, st, group, exchange)

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
        if self.exchange == "peer" and self.world > 1:
            ex = self._peer.get(w)
            if ex is None:
                ex = self._peer[w] = PeerExchange.over_group(self, w)
            return ex.matvec(self.stages, u_local.reshape(ny, self.n1, inner)).reshape(ny * self.n1 * self.n0, w)
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


class NativeComm:
    """An NCCL communicator owned by libtoepcuda over the ranks of a torch.distributed group
    (toep_comm_create; the unique id travels through the group once).  Used by the native
    distributed GMRES: the library enqueues the matvec's all-to-alls and the inner products'
    all-reduce itself."""

    def __init__(self, group=None):
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        lib = _lib.lib()
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _lib.check(lib.toep_comm_unique_id(uid), "comm_unique_id")
        if self.world > 1:
            box = [uid.raw if self.rank == 0 else None]
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            ctypes.memmove(uid, box[0], 128)
        h = ctypes.c_void_p()
        _lib.check(lib.toep_comm_create(uid, self.world, self.rank, ctypes.byref(h)), "comm_create")
        self.handle = h.value

    def check(self):
        """Raise CudaError if NCCL reported an asynchronous error on this communicator."""
        _lib.check(_lib.lib().toep_comm_check(self.handle), "nccl")

    def close(self):
        if getattr(self, "handle", None):
            _lib.lib().toep_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


_COMMS: dict = {}


def native_comm(group=None) -> NativeComm:
    """The library communicator of ``group`` (created once per group, collectively)."""
    key = id(group)
    c = _COMMS.get(key)
    if c is None:
        c = _COMMS[key] = NativeComm(group)
    return c


def gmres_slab(op: SlabOperator, p, b_local, cfg, native: bool | None = None):
    """GMRES (gmres.py:98-249 semantics) on row-distributed vectors of a SlabOperator.

    The device Arnoldi engine (toep_gmres) runs on every rank over the local rows; the
    matvec is the distributed one (two all-to-alls), every inner product and norm is
    all-reduced over the group on the device stream, so all ranks follow identical scalar
    recurrences (same iterations, same stop step).  ``p``: None or an element-block
    preconditioner (P_K, local to each row block).  Returns this rank's rows of x.

    ``native`` (default: on for the device slab operator with the collective exchange): the
    engine calls the library's distributed matvec (toep_slab_apply: level-1 DFT, NCCL
    all-to-all, slab step, all-to-all, inverse level-1 DFT) and NCCL all-reduce directly
    through C function pointers — no Python callback per Arnoldi step.  Otherwise the matvec
    and the all-reduce are Python callbacks (``op.matvec_local``, ``dist.all_reduce``).
    """
    from .solvers.gmres import NativeFn, _run
    from .errors import NoConvergence
    from ._tensor import to_columns, restore

    b, origin = to_columns(b_local)
    if b.shape[0] != op.local_dim:
        raise ShapeError(f"local rhs rows {b.shape[0]} != {op.local_dim}")
    group = op.group
    world = op.world
    auto = native is None
    if auto:
        native = (op.exchange == "collective" and isinstance(op.stages, DeviceSlabStages)
                  and (world == 1 or dist.get_backend(group) == "nccl"))
    comm = None
    if native:
        try:
            comm = native_comm(group)
        except Exception:  # noqa: BLE001 - no usable libnccl: the Python exchange path below
            if not auto:
                raise
            native = False
    if native:
        ctx = ctypes.c_void_p()
        _lib.check(_lib.lib().toep_slab_ctx_create(op.stages.op.handle, comm.handle, b.shape[1],
                                                   _lib.stream_handle(), ctypes.byref(ctx)), "slab_ctx_create")
        try:
            x, report = _run(NativeFn("toep_slab_apply", ctx.value), p, b, cfg, prefer_numpy=False,
                             allreduce=NativeFn("toep_comm_allreduce", comm.handle))
        finally:
            _lib.lib().toep_slab_ctx_destroy(ctx.value)
        comm.check()
        report.method = "gmres-slab"
        xo = restore(x, origin)
        if not report.converged:
            raise NoConvergence(f"distributed GMRES stopped after {report.iterations} iterations", solution=xo,
                                report=report)
        return xo, report

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
    """The three local stages of SlabOperator on the device (toep_matvec_stage).

    The rank's slab operator is built straight from the generator (``toep_op_create_slab``): the
    level-2 DFT runs only over the rank's level-1 frequencies, so no rank ever holds the full
    spectral operator (resident bytes = D * kxs / l1).  ``gen`` may be a generator, a host stacked
    array or a CUDA tensor of the stacked blocks (e.g. broadcast from rank 0).
    """

    def __init__(self, gen, world: int, rank: int, dtype, embedding=None):
        from .toeplitz import _smooth7, precompute_spectral_stacked

        stacked = gen if isinstance(gen, (np.ndarray, torch.Tensor)) else gen.stacked4()
        k2, k1, n0 = int(stacked.shape[0]), int(stacked.shape[1]), int(stacked.shape[2])
        self.n2, self.n1, self.n0 = (k2 + 1) // 2, (k1 + 1) // 2, n0
        self.l2, self.l1 = embedding if embedding is not None else (_smooth7(k2), _smooth7(k1))
        k0, k1_ = slab_ranges(self.l1, world, rank)
        self.op = precompute_spectral_stacked(stacked, dtype=dtype, embedding=(self.l2, self.l1), slab=(k0, k1_))
        self.k0, self.k1 = k0, k1_

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

    # peer mode: stages 0 / 1 store into the destination ranks' receive buffers (table: device
    # toep_peer_scatter built by PeerExchange) and signal their arrival counters
    def _stage_peer(self, stage: int, x: torch.Tensor, table: torch.Tensor, count: int):
        x = x.contiguous()
        w = x.shape[-1] // self.n0
        _lib.check(_lib.lib().toep_matvec_stage_peer(self.op.handle, stage, x.data_ptr(), table.data_ptr(), w, count,
                                                     _lib.stream_handle()), f"matvec_stage_peer {stage}")

    def fwd_x_peer(self, u_rows, table):
        self._stage_peer(0, u_rows, table, u_rows.shape[0])

    def spectral_peer(self, x1_slab, table):
        self._stage_peer(1, x1_slab, table, x1_slab.shape[1])


def scatter_plan(stage: int, rank: int, world: int, n2: int, l1: int, inner: int):
    """Routing of one peer-scatter pass of ``rank`` (elements of each destination's buffer).

    stage 0 — level-1 DFT of this rank's rows; output index = kx, outer index o = local row.
        Destination q's receive buffer 1 is (n2, kxs_q, inner): element (y0_r + o, kx - k0_q, i).
    stage 1 — inverse level-2 DFT of this rank's kx slab; output index = y, outer o = local kx.
        Destination q's receive buffer 2 is (ny_q, l1, inner): element (y - y0_q, k0_r + o, i).
    Returns ``(lo, parts)``: output index range [lo[q], lo[q+1]) goes to q at
    ``off + a*sa + o*so + i`` with ``parts[q] = (off, sa, so)`` — the C table's fields.
    """
    if not 1 <= world <= _lib.MAX_PEERS:
        raise ValueError(f"peer exchange supports 1..{_lib.MAX_PEERS} ranks, got {world}")
    if world > n2 or world > l1:  # every rank must own rows and a slab: each pass signals every peer
        raise ShapeError(f"peer exchange needs world ({world}) <= rows ({n2}) and <= level-1 length ({l1})")
    rows = [row_range(n2, world, q) for q in range(world)]
    slabs = [slab_ranges(l1, world, q) for q in range(world)]
    y0, _ = rows[rank]
    k0, _ = slabs[rank]
    if stage == 0:
        lo = [a for a, _ in slabs] + [l1]
        parts = [((y0 * (b - a) - a) * inner, inner, (b - a) * inner) for a, b in slabs]
    elif stage == 1:
        lo = [a for a, _ in rows] + [n2]
        parts = [((-a * l1 + k0) * inner, l1 * inner, inner) for a, _ in rows]
    else:
        raise ValueError(f"peer scatter is defined for stages 0 and 1, not {stage}")
    return lo, parts


class PeerExchange:
    """Receive buffers + arrival counters of one rank, mapped into every peer (CUDA IPC).

    One ``cudaMalloc`` region per rank and column count w: two u64 arrival counters, receive
    buffer 1 (n2, kxs_r, n0*w) and receive buffer 2 (ny_r, l1, n0*w).  ``tables`` are the device
    routing tables of this rank's two scatter passes (``scatter_plan`` resolved to the peers'
    mapped addresses).  A matvec: stage 0 scatters to the slab owners, wait for ``world`` arrivals
    on counter 1, stage 1 on receive buffer 1 scatters to the row owners, wait on counter 2,
    stage 2 on receive buffer 2.  Buffer reuse across matvecs is safe by construction: a rank
    writes a peer's buffer for matvec m+1 only after that peer has signalled the exchange that
    follows its last read of it in matvec m.
    """

    _HDR = 256

    def __init__(self, sizes, es: int, device):
        self.es = es
        self.device = device
        self.seq = 0
        self.world = None
        n1b, n2b = sizes
        self.off1 = self._HDR
        self.off2 = self._HDR + -(-n1b * es // 256) * 256
        self.bytes = self.off2 + n2b * es
        ptr = ctypes.c_void_p()
        _lib.check(_lib.lib().toep_peer_alloc(self.bytes, ctypes.byref(ptr)), "peer_alloc")
        self.base = ptr.value
        self.sizes = sizes
        self._opened = []
        self.tables = None

    @staticmethod
    def _sizes(op: "SlabOperator", rank: int, w: int):
        inner = op.n0 * w
        y0, y1 = row_range(op.n2, op.world, rank)
        k0, k1 = slab_ranges(op.l1, op.world, rank)
        return op.n2 * (k1 - k0) * inner, (y1 - y0) * op.l1 * inner

    @classmethod
    def over_group(cls, op: "SlabOperator", w: int) -> "PeerExchange":
        """Collective setup over op.group: allocate, exchange IPC handles, open the peers."""
        es = 8 if op.stages.op.dtype == torch.complex64 else 16
        ex = cls(cls._sizes(op, op.rank, w), es, torch.device("cuda", torch.cuda.current_device()))
        h = (ctypes.c_char * 64)()
        _lib.check(_lib.lib().toep_ipc_handle(ctypes.c_void_p(ex.base), h), "ipc_handle")
        mine = (bytes(h), ex.off1, ex.off2)
        got = [None] * op.world
        dist.all_gather_object(got, mine, group=op.group)
        bases = []
        for q, (hq, _, _) in enumerate(got):
            if q == op.rank:
                bases.append(ex.base)
                continue
            p = ctypes.c_void_p()
            _lib.check(_lib.lib().toep_ipc_open(ctypes.create_string_buffer(hq, 64), ctypes.byref(p)), "ipc_open")
            ex._opened.append(p.value)
            bases.append(p.value)
        ex.bind(op.rank, op.world, op.n2, op.l1, op.n0 * w,
                [(b, g[1], g[2]) for b, g in zip(bases, got)])
        return ex

    def bind(self, rank: int, world: int, n2: int, l1: int, inner: int, peers):
        """Build this rank's two device routing tables; peers[q] = (base address, off1, off2)."""
        self.world, self.rank = world, rank
        tables = []
        for stage, (sig_off, buf) in ((0, (0, 1)), (1, (8, 2))):
            lo, parts = scatter_plan(stage, rank, world, n2, l1, inner)
            t = _lib.PeerScatter()
            t.parts = world
            for q in range(world + 1):
                t.lo[q] = lo[q]
            for q, (off, sa, so) in enumerate(parts):
                base_q, o1, o2 = peers[q]
                t.base[q] = base_q + (o1 if buf == 1 else o2)
                t.off[q], t.sa[q], t.so[q] = off, sa, so
                t.signal[q] = base_q + sig_off
            t.done = 0
            raw = torch.frombuffer(bytearray(bytes(t)), dtype=torch.uint8)
            tables.append(raw.to(self.device))
        self.tables = tables

    def recv(self, which: int, shape, dtype):
        """Device tensor view of receive buffer 1 or 2 (owned by this object)."""
        off, n = (self.off1, self.sizes[0]) if which == 1 else (self.off2, self.sizes[1])
        return _device_view(self.base + off, n, dtype, self.device).reshape(shape)

    def counter(self, which: int) -> int:
        return self.base + (0 if which == 1 else 8)

    def wait(self, which: int, stream=None):
        _lib.check(_lib.lib().toep_peer_wait(ctypes.c_void_p(self.counter(which)), self.seq * self.world,
                                             stream if stream is not None else _lib.stream_handle()), "peer_wait")

    def matvec(self, stages: "DeviceSlabStages", u_rows: torch.Tensor) -> torch.Tensor:
        """One distributed matvec of this rank's rows (ny_r, n1, n0*w) -> (ny_r, n1, n0*w)."""
        ny, _, inner = u_rows.shape
        dtype = stages.op.dtype
        kxs = stages.k1 - stages.k0
        self.seq += 1
        stages.fwd_x_peer(u_rows, self.tables[0])
        self.wait(1)
        stages.spectral_peer(self.recv(1, (stages.n2, kxs, inner), dtype), self.tables[1])
        self.wait(2)
        return stages.inv_x(self.recv(2, (ny, stages.l1, inner), dtype))

    def close(self):
        lib = _lib.lib()
        for p in self._opened:
            lib.toep_ipc_close(ctypes.c_void_p(p))
        self._opened = []
        if self.base:
            lib.toep_peer_free(ctypes.c_void_p(self.base))
            self.base = 0

    def __del__(self):
        try:
            if torch.cuda.is_available():
                torch.cuda.synchronize(self.device)
            self.close()
        except Exception:
            pass


def _device_view(addr: int, numel: int, dtype, device) -> torch.Tensor:
    """Non-owning torch view of device memory allocated by libtoepcuda."""
    es = torch.empty((), dtype=dtype).element_size()

    class _Mem:
        __cuda_array_interface__ = {"shape": (numel * es,), "typestr": "|u1", "data": (addr, False), "version": 3}

    return torch.as_tensor(_Mem(), device=device).view(dtype)
