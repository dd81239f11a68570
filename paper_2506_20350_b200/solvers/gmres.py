"""Left-preconditioned GMRES (drop-in for solvers/gmres.py of the reference).

The iteration itself runs inside ``libtoepcuda`` (``toep_gmres``): Krylov
basis, Hessenberg columns, Givens rotations, residual history and stop flags
are device resident and the host thread only launches work, one Arnoldi step
ahead of the device.  Semantics are those of ``_gmres_block``
(gmres.py:98-219): Frobenius inner products over (n, W) blocks (global Krylov
for W > 1), full GMRES unless ``restart``, relative *preconditioned* residual
history from the Givens recurrence, true unpreconditioned residual at exit,
``NoConvergence`` carrying the iterate and report.

Dispatch:
  * operator = ``BorderedOperator`` (no border) / ``SpectralOperator``: the
    matvec is called natively; an element preconditioner (PK) is folded into
    the operator (D_k <- R_00^-1 D_k, computed once and cached);
  * any other callable: called back from the device loop with CUDA tensors
    (or numpy arrays, if the callable rejects tensors), results copied back.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .. import _lib
from .._tensor import Origin, restore, to_columns
from ..errors import NoConvergence, ShapeError
from ..toeplitz import SpectralOperator
from .bordered import BorderedOperator, bordered_matvec
from .precond import Preconditioner, apply_precond

__all__ = [
    "GmresConfig",
    "SolveReport",
    "gmres",
    "solve_multi_rhs_vectorized",
    "solve_multi_rhs_sequential",
]

_BYTES_PER_SCALAR = 16


@dataclass
class GmresConfig:
    tol: float = 1e-3
    max_iter: int = 500
    restart: int | None = None

    def __post_init__(self):
        if not self.tol > 0:
            raise ValueError(f"tol must be > 0, got {self.tol}")
        if self.max_iter < 1:
            raise ValueError(f"max_iter must be >= 1, got {self.max_iter}")
        if self.restart is not None and self.restart < 1:
            raise ValueError(f"restart must be >= 1, got {self.restart}")


def _new_timings() -> dict:
    return {"precond_build": 0.0, "precond_apply": 0.0, "matvec_total": 0.0, "orthogonalization": 0.0,
            "total": 0.0}


def _new_memory() -> dict:
    return {"generator": 0, "krylov": 0, "preconditioner": 0}


@dataclass
class SolveReport:
    """Bookkeeping of one solve (gmres.py:63-84)."""

    method: str = ""
    iterations: int = 0
    converged: bool = True
    residual_history: list = field(default_factory=list)
    final_residual: float = 0.0
    phase_timings: dict = field(default_factory=_new_timings)
    memory_estimate: dict = field(default_factory=_new_memory)

    def as_dict(self) -> dict:
        return {
            "method": self.method,
            "iterations": self.iterations,
            "converged": self.converged,
            "residual_history": list(self.residual_history),
            "final_residual": self.final_residual,
            "phase_timings": dict(self.phase_timings),
            "memory_estimate": dict(self.memory_estimate),
        }


class _CallablePrecond:
    def __init__(self, fn):
        self.fn = fn

    def apply(self, v):
        return self.fn(v)


def _coerce_precond(p):
    if p is None or hasattr(p, "apply"):
        return p
    if callable(p):
        return _CallablePrecond(p)
    raise TypeError(f"cannot use {type(p).__name__} as a preconditioner")


def _native_op(op):
    """SpectralOperator behind ``op`` when the fast path applies, else None."""
    if isinstance(op, SpectralOperator):
        return op
    if isinstance(op, BorderedOperator) and op.nb == 0:
        return op.spectral
    return None


_FOLD_CACHE: dict = {}


def _fold_cached(spec: SpectralOperator, p: Preconditioner) -> bool:
    hit = _FOLD_CACHE.get((id(spec), id(p)))
    return hit is not None and hit[0] is spec and hit[1] is p


def _folded(spec: SpectralOperator, p: Preconditioner) -> SpectralOperator:
    key = (id(spec), id(p))
    hit = _FOLD_CACHE.get(key)
    if hit is not None and hit[0] is spec and hit[1] is p:
        return hit[2]
    folded = spec.fold_left(p.device_blocks()["pinv"])
    _FOLD_CACHE.clear()  # keep at most one folded copy resident
    _FOLD_CACHE[key] = (spec, p, folded)
    return folded


class _DeviceView:
    def __init__(self, ptr: int, n: int, w: int):
        self.__cuda_array_interface__ = {"shape": (n, w), "typestr": "<c16", "data": (ptr, False),
                                         "version": 3, "strides": None}


class _Callback:
    """Adapter from the C callback (x ptr -> y ptr) to a Python callable."""

    def __init__(self, fn, n: int, w: int, prefer_numpy: bool):
        self.fn = fn
        self.n, self.w = n, w
        self.mode = "numpy" if prefer_numpy else "torch"
        self.error = None
        self.cfunc = _lib.APPLY_FN(self._call)

    def _invoke(self, x: torch.Tensor):
        if self.mode == "torch":
            try:
                out = self.fn(x)
                if isinstance(out, torch.Tensor):
                    return out
                return torch.as_tensor(np.asarray(out), device=x.device)
            except (TypeError, RuntimeError, ValueError):
                self.mode = "numpy"
        out = self.fn(x.cpu().numpy())
        if isinstance(out, torch.Tensor):
            return out.to(x.device)
        return torch.from_numpy(np.ascontiguousarray(np.asarray(out, dtype=np.complex128))).to(x.device)

    def _call(self, ctx, xptr, yptr, w, stream):
        try:
            dev = torch.device("cuda", torch.cuda.current_device())
            x = torch.as_tensor(_DeviceView(xptr, self.n, w), device=dev)
            y = torch.as_tensor(_DeviceView(yptr, self.n, w), device=dev)
            out = self._invoke(x)
            y.copy_(out.reshape(self.n, w).to(torch.complex128))
            return 0
        except BaseException as exc:  # noqa: BLE001 - re-raised after the C call returns
            self.error = exc
            return 1


class _AllReduce:
    """C callback: sum a device float64 buffer over the process group (NCCL, stream ordered)."""

    def __init__(self, fn):
        self.fn = fn
        self.error = None
        self.cfunc = _lib.ALLREDUCE_FN(self._call)

    def _call(self, ctx, ptr, ndoubles, stream):
        try:
            dev = torch.device("cuda", torch.cuda.current_device())
            view = {"shape": (ndoubles,), "typestr": "<f8", "data": (ptr, False), "version": 3, "strides": None}
            t = torch.as_tensor(type("V", (), {"__cuda_array_interface__": view})(), device=dev)
            self.fn(t)
            return 0
        except BaseException as exc:  # noqa: BLE001
            self.error = exc
            return 1


class NativeFn:
    """A library function (address) with its context pointer, passed to toep_gmres as the operator
    (toep_apply_fn signature) or the all-reduce (e.g. toep_slab_apply / toep_comm_allreduce): the
    engine calls it directly, no Python in the Arnoldi loop."""

    def __init__(self, name: str, ctx: int):
        self.addr = ctypes.cast(getattr(_lib.lib(), name), ctypes.c_void_p).value
        self.ctx = ctx


def _run(apply_op, precond, b: torch.Tensor, cfg: GmresConfig, prefer_numpy: bool, timings: bool = True,
         allreduce=None):
    """Run toep_gmres on a device (n, w) complex128 block; returns (x, SolveReport).

    ``allreduce(t)``: optional in-place sum of a device float64 tensor over ranks, for
    Krylov vectors distributed by rows (distributed.gmres_slab).
    """
    n, w = b.shape
    prob = _lib.GmresProblem()
    keep = []  # keep ctypes callbacks / tensors alive for the call
    if isinstance(allreduce, NativeFn):
        prob.allreduce = _lib.ALLREDUCE_FN(allreduce.addr)
        prob.allreduce_ctx = allreduce.ctx
    elif allreduce is not None:
        ar = _AllReduce(allreduce)
        prob.allreduce = ar.cfunc
        keep.append(ar)
    native = None if isinstance(apply_op, NativeFn) else _native_op(apply_op)
    report = SolveReport()
    t_build = 0.0
    pc = precond
    if isinstance(pc, Preconditioner) and pc.kind == "none":
        pc = None
    if native is not None:
        if native.dim != n:
            raise ShapeError(f"rhs rows {n} != operator dim {native.dim}")
        if isinstance(pc, Preconditioner) and pc.nb == 0 and pc.kind == "pk" and pc.side == native.n0:
            t0 = time.perf_counter()
            cached = _fold_cached(native, pc)
            folded = _folded(native, pc)
            d = pc.device_blocks()
            if not cached:  # time the fold itself (a cached fold costs nothing and needs no wait)
                torch.cuda.current_stream().synchronize()
            t_build = time.perf_counter() - t0
            prob.op = folded.handle
            prob.precond = _lib.TOEP_PC_FOLDED
            prob.pinv, prob.pmat, prob.pside = d["pinv"].data_ptr(), d["pmat"].data_ptr(), pc.side
            keep += [folded, d]
            pc = "done"
        else:
            prob.op = native.handle
    elif isinstance(apply_op, NativeFn):
        prob.op = None
        prob.apply = _lib.APPLY_FN(apply_op.addr)
        prob.apply_ctx = apply_op.ctx
    else:
        cb = _Callback(apply_op, n, w, prefer_numpy)
        prob.op = None
        prob.apply = cb.cfunc
        keep.append(cb)
    if pc != "done":
        if pc is None:
            prob.precond = _lib.TOEP_PC_NONE
        elif isinstance(pc, Preconditioner) and pc.nb == 0:
            d = pc.device_blocks()
            prob.precond = _lib.TOEP_PC_BLOCK
            prob.pinv, prob.pside = d["pinv"].data_ptr(), pc.side
            keep.append(d)
        else:
            pcb = _Callback(lambda v: pc.apply(v), n, w, prefer_numpy)
            prob.precond = _lib.TOEP_PC_CALLBACK
            prob.papply = pcb.cfunc
            keep.append(pcb)
    prob.n, prob.w = n, w
    max_total = min(cfg.max_iter, n * w)
    hist = np.zeros(max_total + 2, dtype=np.float64)
    rep = _lib.GmresReport()
    rep.history = hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    rep.history_cap = hist.size
    c = _lib.GmresCfg(float(cfg.tol), int(cfg.max_iter), int(cfg.restart or 0), int(timings))
    x = torch.empty_like(b)
    status = _lib.lib().toep_gmres(ctypes.byref(prob), ctypes.byref(c), b.data_ptr(), x.data_ptr(),
                                   _lib.stream_handle(), ctypes.byref(rep))
    for k in keep:
        err = getattr(k, "error", None)
        if err is not None:
            raise err
    _lib.check(status, "gmres")
    report.iterations = int(rep.iterations)
    report.converged = bool(rep.converged)
    report.residual_history = hist[: rep.n_history].tolist()
    report.final_residual = float(rep.final_residual)
    report.phase_timings.update(precond_build=t_build, precond_apply=rep.t_precond, matvec_total=rep.t_matvec,
                                orthogonalization=rep.t_orth, total=rep.t_total + t_build)
    report.memory_estimate["krylov"] = report.iterations * w * n * _BYTES_PER_SCALAR
    return x, report


def gmres(apply_operator, apply_precond_fn, rhs, cfg: GmresConfig):
    """Solve A x = b with left-preconditioned GMRES (gmres.py:222-249)."""
    b, origin = to_columns(rhs)
    if b.ndim != 2:
        raise ShapeError("rhs must be 1-D or 2-D")
    pre = _coerce_precond(apply_precond_fn)
    x, report = _run(apply_operator, pre, b, cfg, prefer_numpy=False)
    xo = restore(x, origin)
    if not report.converged:
        raise NoConvergence(
            f"GMRES stopped after {report.iterations} iterations at relative preconditioned residual "
            f"{report.residual_history[-1]:.3e} > tol {cfg.tol:.1e}", solution=xo, report=report)
    return xo, report


def _operator_memory(op, p, report: SolveReport) -> None:
    if isinstance(op, BorderedOperator):
        report.memory_estimate["generator"] = op.generator_bytes
    if p is not None and hasattr(p, "stored_bytes"):
        report.memory_estimate["preconditioner"] = p.stored_bytes


def _as_block(rhs):
    if isinstance(rhs, torch.Tensor):
        if rhs.ndim != 2:
            raise ShapeError(f"rhs must be a column block, got ndim={rhs.ndim}")
    else:
        if np.ndim(rhs) != 2:
            raise ShapeError(f"rhs must be a column block, got ndim={np.ndim(rhs)}")
    return to_columns(rhs)


def solve_multi_rhs_vectorized(op, p, rhs, cfg: GmresConfig, method: str = "vectorized"):
    """One global-Krylov GMRES over all columns jointly (gmres.py:275-301)."""
    b, origin = _as_block(rhs)
    apply_op = op
    if _native_op(op) is None and not callable(op):
        apply_op = lambda x: bordered_matvec(op, x)  # noqa: E731
    pre = _coerce_precond(p)
    t0 = time.perf_counter()
    x, report = _run(apply_op, pre, b, cfg, prefer_numpy=False)
    report.method = method
    report.phase_timings["total"] = time.perf_counter() - t0
    _operator_memory(op, p, report)
    xo = restore(x, origin)
    if not report.converged:
        raise NoConvergence(f"vectorized GMRES stopped after {report.iterations} iterations above tol",
                            solution=xo, report=report)
    return xo, report


def _run_batched(native: SpectralOperator, pc, b: torch.Tensor, cfg: GmresConfig, method: str):
    """All columns through toep_gmres_batched (lock-step independent solves)."""
    n, w = b.shape
    prob = _lib.GmresProblem()
    keep = []
    t_build = 0.0
    if pc is None or (isinstance(pc, Preconditioner) and pc.kind == "none"):
        prob.op = native.handle
        prob.precond = _lib.TOEP_PC_NONE
    elif pc.kind == "pk" and pc.side == native.n0:
        t0 = time.perf_counter()
        cached = _fold_cached(native, pc)
        folded = _folded(native, pc)
        d = pc.device_blocks()
        if not cached:
            torch.cuda.current_stream().synchronize()
        t_build = time.perf_counter() - t0
        prob.op = folded.handle
        prob.precond = _lib.TOEP_PC_FOLDED
        prob.pinv, prob.pmat, prob.pside = d["pinv"].data_ptr(), d["pmat"].data_ptr(), pc.side
        keep += [folded, d]
    else:
        d = pc.device_blocks()
        prob.op = native.handle
        prob.precond = _lib.TOEP_PC_BLOCK
        prob.pinv, prob.pside = d["pinv"].data_ptr(), pc.side
        keep.append(d)
    prob.n, prob.w = n, w
    max_total = min(cfg.max_iter, n)
    rows = max_total + 2
    iters = np.zeros(w, dtype=np.int32)
    conv = np.zeros(w, dtype=np.int32)
    final = np.zeros(w, dtype=np.float64)
    nhist = np.zeros(w, dtype=np.int32)
    hist = np.zeros((rows, w), dtype=np.float64)
    c = _lib.GmresCfg(float(cfg.tol), int(cfg.max_iter), int(cfg.restart or 0), 0)
    x = torch.empty_like(b)
    t0 = time.perf_counter()
    _lib.check(_lib.lib().toep_gmres_batched(ctypes.byref(prob), ctypes.byref(c), b.data_ptr(), x.data_ptr(),
                                             _lib.stream_handle(), iters.ctypes.data, conv.ctypes.data,
                                             final.ctypes.data, nhist.ctypes.data, hist.ctypes.data, rows),
               "gmres_batched")
    total = time.perf_counter() - t0 + t_build
    reports = []
    for col in range(w):
        rep = SolveReport(method=method, iterations=int(iters[col]), converged=bool(conv[col]),
                          residual_history=hist[: nhist[col], col].tolist(), final_residual=float(final[col]))
        rep.phase_timings.update(precond_build=t_build, total=total)
        rep.memory_estimate["krylov"] = rep.iterations * n * _BYTES_PER_SCALAR
        reports.append(rep)
    return x, reports


def solve_multi_rhs_sequential(op, p, rhs, cfg: GmresConfig, method: str = "sequential"):
    """Independent GMRES per column (gmres.py:304-336).

    With a resident operator the columns run as one lock-step batch
    (``toep_gmres_batched``): every Arnoldi step is one multi-RHS matvec whose
    per-bin product is a tensor-core complex GEMM; each column keeps its own
    Krylov space, rotations, history and stop flag, so its iterate and report
    are those of an independent solve.
    """
    b, origin = _as_block(rhs)
    native = _native_op(op)
    pre = _coerce_precond(p)
    if native is not None and (pre is None or (isinstance(pre, Preconditioner) and pre.nb == 0)):
        if native.dim != b.shape[0]:
            raise ShapeError(f"rhs rows {b.shape[0]} != operator dim {native.dim}")
        x, reports = _run_batched(native, pre, b, cfg, method)
        for rep in reports:
            _operator_memory(op, p, rep)
        xo = restore(x, origin)
        failed = [c for c, r in enumerate(reports) if not r.converged]
        if failed:
            raise NoConvergence(f"columns {failed} did not converge within {cfg.max_iter} iterations",
                                solution=xo, reports=reports)
        return xo, reports
    apply_op = op
    if _native_op(op) is None and not callable(op):
        apply_op = lambda x: bordered_matvec(op, x)  # noqa: E731
    pre = _coerce_precond(p)
    x = torch.empty_like(b)
    reports = []
    failed = []
    for col in range(b.shape[1]):
        xi, rep = _run(apply_op, pre, b[:, col:col + 1].contiguous(), cfg, prefer_numpy=False)
        rep.method = method
        _operator_memory(op, p, rep)
        x[:, col] = xi[:, 0]
        reports.append(rep)
        if not rep.converged:
            failed.append(col)
    xo = restore(x, origin)
    if failed:
        raise NoConvergence(f"columns {failed} did not converge within {cfg.max_iter} iterations",
                            solution=xo, reports=reports)
    return xo, reports
