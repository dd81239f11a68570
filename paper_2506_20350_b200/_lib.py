"""ctypes binding of libtoepcuda.so (the C ABI declared in include/toepcuda.h).

The shared library is built in-tree (``paper_2506_20350_b200/libtoepcuda.so``,
see ``csrc/Makefile`` / ``__graft_entry__.build``).  There is no CPU fallback:
if the library or a CUDA device is missing every device entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TOEPCUDA_LIB", os.path.join(_HERE, "libtoepcuda.so"))

TOEP_OK = 0
TOEP_ERR_SHAPE = 1
TOEP_ERR_ARG = 2
TOEP_ERR_SINGULAR = 3
TOEP_ERR_SINGULAR_BLOCK = 4
TOEP_ERR_SINGULAR_DENOM = 5
TOEP_ERR_NOCONV = 6
TOEP_ERR_CUDA = 7
TOEP_ERR_OOM = 8

TOEP_C128 = 0
TOEP_C64 = 1

TOEP_MV_TRANSPOSE = 1
TOEP_MV_IO_C128 = 2
TOEP_MV_STAGE_INPUT = 4

TOEP_PC_NONE = 0
TOEP_PC_BLOCK = 1
TOEP_PC_FOLDED = 2
TOEP_PC_CALLBACK = 3

c_int = ctypes.c_int
c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_vp = ctypes.c_void_p
c_dbl = ctypes.c_double

APPLY_FN = ctypes.CFUNCTYPE(c_int, c_vp, c_vp, c_vp, c_i64, c_vp)
STAGE_FN = ctypes.CFUNCTYPE(c_int, c_vp, c_int, c_vp, c_vp, c_vp, c_vp)
ALLREDUCE_FN = ctypes.CFUNCTYPE(c_int, c_vp, c_vp, c_i64, c_vp)


class OpInfo(ctypes.Structure):
    _fields_ = [("n2", c_i32), ("n1", c_i32), ("n0", c_i32), ("l2", c_i32), ("l1", c_i32), ("dtype", c_i32),
                ("bins", c_i64), ("dim", c_i64), ("resident_bytes", c_i64)]


MAX_PEERS = 8


class PeerScatter(ctypes.Structure):
    """toep_peer_scatter (include/toepcuda.h): output-row routing table of a peer-scatter pass."""
    _fields_ = [("parts", c_i64), ("lo", c_i64 * (MAX_PEERS + 1)), ("base", ctypes.c_uint64 * MAX_PEERS),
                ("off", c_i64 * MAX_PEERS), ("sa", c_i64 * MAX_PEERS), ("so", c_i64 * MAX_PEERS),
                ("signal", ctypes.c_uint64 * MAX_PEERS), ("done", ctypes.c_uint64)]


class GmresProblem(ctypes.Structure):
    _fields_ = [("op", c_vp), ("apply", APPLY_FN), ("apply_ctx", c_vp), ("precond", c_i32), ("pside", c_i32),
                ("pinv", c_vp), ("pmat", c_vp), ("papply", APPLY_FN), ("papply_ctx", c_vp),
                ("n", c_i64), ("w", c_i64), ("allreduce", ALLREDUCE_FN), ("allreduce_ctx", c_vp)]


class GmresCfg(ctypes.Structure):
    _fields_ = [("tol", c_dbl), ("max_iter", c_i32), ("restart", c_i32), ("timings", c_i32)]


class GmresReport(ctypes.Structure):
    _fields_ = [("iterations", c_i32), ("converged", c_i32), ("breakdown", c_i32), ("n_history", c_i32),
                ("final_residual", c_dbl), ("t_matvec", c_dbl), ("t_precond", c_dbl), ("t_orth", c_dbl),
                ("t_total", c_dbl), ("history", ctypes.POINTER(c_dbl)), ("history_cap", c_i32)]


# name -> (restype, argtypes); every symbol include/toepcuda.h declares
SIGNATURES = {
    "toep_last_error": (ctypes.c_char_p, []),
    "toep_version": (c_int, []),
    "toep_fnv1a64": (c_int, [c_vp, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]),
    "toep_op_create": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_vp, ctypes.POINTER(c_vp)]),
    "toep_op_destroy": (c_int, [c_vp]),
    "toep_op_info": (c_int, [c_vp, ctypes.POINTER(OpInfo)]),
    "toep_op_diag_blocks": (c_int, [c_vp, c_vp, c_vp]),
    "toep_op_fold_left": (c_int, [c_vp, c_vp, c_vp, ctypes.POINTER(c_vp)]),
    "toep_matvec": (c_int, [c_vp, c_vp, c_vp, c_i64, c_int, c_vp]),
    "toep_matvec_host": (c_int, [c_vp, c_vp, c_vp, c_i64, c_int, c_vp]),
    "toep_host_alloc": (c_int, [ctypes.c_uint64, ctypes.POINTER(c_vp)]),
    "toep_h2d": (c_int, [c_vp, c_vp, ctypes.c_uint64, c_vp]),
    "toep_ozaki_dgemm": (c_int, [c_int, c_int, c_i64, ctypes.c_double, c_vp, c_i64, c_vp, c_i64, ctypes.c_double, c_vp,
                                 c_i64, c_vp]),
    "toep_comm_unique_id": (c_int, [c_vp]),
    "toep_comm_create": (c_int, [c_vp, c_int, c_int, ctypes.POINTER(c_vp)]),
    "toep_comm_destroy": (c_int, [c_vp]),
    "toep_comm_check": (c_int, [c_vp]),
    "toep_comm_allreduce": (c_int, [c_vp, c_vp, c_i64, c_vp]),
    "toep_slab_ctx_create": (c_int, [c_vp, c_vp, c_i64, c_vp, ctypes.POINTER(c_vp)]),
    "toep_slab_ctx_destroy": (c_int, [c_vp]),
    "toep_slab_apply": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "toep_host_free": (c_int, [c_vp]),
    "toep_op_slab": (c_int, [c_vp, c_int, c_int, c_vp, ctypes.POINTER(c_vp)]),
    "toep_op_create_slab": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_vp,
                                    ctypes.POINTER(c_vp)]),
    "toep_matvec_stage": (c_int, [c_vp, c_int, c_vp, c_vp, c_i64, c_int, c_vp]),
    "toep_matvec_stage_peer": (c_int, [c_vp, c_int, c_vp, c_vp, c_i64, c_int, c_vp]),
    "toep_peer_wait": (c_int, [c_vp, ctypes.c_uint64, c_vp]),
    "toep_peer_alloc": (c_int, [ctypes.c_uint64, ctypes.POINTER(c_vp)]),
    "toep_peer_free": (c_int, [c_vp]),
    "toep_ipc_handle": (c_int, [c_vp, c_vp]),
    "toep_ipc_open": (c_int, [c_vp, ctypes.POINTER(c_vp)]),
    "toep_ipc_close": (c_int, [c_vp]),
    "toep_op_spectral_apply": (c_int, [c_vp, c_vp, c_vp, c_i64, c_int, c_vp]),
    "toep_block_dft": (c_int, [c_vp, c_vp, c_int, c_int, c_i64, c_int, c_int, c_vp]),
    "toep_block_apply": (c_int, [c_vp, c_int, c_vp, c_vp, c_i64, c_i64, c_int, c_vp]),
    "toep_gemm": (c_int, [c_int, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_i64, c_i64,
                          c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp]),
    "toep_dgemm": (c_int, [c_i64, c_i64, c_i64, c_dbl, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_i64, c_i64, c_dbl,
                           c_vp, c_i64, c_i64, c_i64, c_i64, c_vp]),
    "toep_gmres": (c_int, [ctypes.POINTER(GmresProblem), ctypes.POINTER(GmresCfg), c_vp, c_vp, c_vp,
                           ctypes.POINTER(GmresReport)]),
    "toep_lu_factor": (c_int, [c_vp, c_int, c_vp, c_vp, c_vp]),
    "toep_lu_solve": (c_int, [c_vp, c_int, c_vp, c_vp, c_i64, c_vp]),
    "toep_rybicki": (c_int, [c_vp, c_int, c_int, c_vp, c_vp, c_i64, ctypes.POINTER(c_int), c_vp, c_vp, c_vp]),
    "toep_assemble_level1": (c_int, [c_vp, c_int, c_int, c_int, c_vp, c_vp]),
    "toep_gmres_batched": (c_int, [ctypes.POINTER(GmresProblem), ctypes.POINTER(GmresCfg), c_vp, c_vp, c_vp,
                                   c_vp, c_vp, c_vp, c_vp, c_vp, c_i64]),
}

_lib = None
_lock = threading.Lock()


def load(path: str | None = None):
    """Load (once) and return the CDLL; raises if the library is absent."""
    global _lib
    with _lock:
        if _lib is None:
            p = path or LIB_PATH
            if not os.path.exists(p):
                raise RuntimeError(
                    f"libtoepcuda.so not found at {p}; build it with `python -c 'import __graft_entry__ as g; "
                    "g.build()'` (or `make -C paper_2506_20350_b200/csrc`). There is no CPU fallback.")
            lib = ctypes.CDLL(p)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def lib():
    return _lib if _lib is not None else load()


_CUDA_OK = False
_DEVICES: dict = {}


def require_cuda() -> torch.device:
    global _CUDA_OK
    if not _CUDA_OK:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2506_20350_b200 needs a CUDA device (B200 / sm_100a); no CPU fallback exists")
        lib()
        _CUDA_OK = True
    idx = torch.cuda.current_device()
    dev = _DEVICES.get(idx)
    if dev is None:
        dev = _DEVICES[idx] = torch.device("cuda", idx)
    return dev


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle(stream=None) -> int:
    """cudaStream_t of ``stream`` (default: torch's current stream on the current device)."""
    if stream is not None:
        return int(stream.cuda_stream)
    if _raw_stream is not None:  # skips building a torch.cuda.Stream object per call
        return int(_raw_stream(torch.cuda.current_device()))
    return int(torch.cuda.current_stream().cuda_stream)


def upload(arr, dev) -> torch.Tensor:
    """A C-contiguous numpy array copied to a new tensor on CUDA device ``dev`` through the
    library's staged page-locked path (toep_h2d), ordered on torch's current stream."""
    import numpy as np

    a = np.ascontiguousarray(arr)
    out = torch.empty(a.shape, dtype=torch.from_numpy(a[:0].reshape(-1)).dtype, device=dev)
    if a.nbytes:
        check(lib().toep_h2d(a.ctypes.data, out.data_ptr(), a.nbytes, stream_handle()), "upload")
    return out


def last_error() -> str:
    msg = lib().toep_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(status: int, what: str = "") -> None:
    if status == TOEP_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == TOEP_ERR_SHAPE:
        raise errors.ShapeError(msg)
    if status == TOEP_ERR_ARG:
        raise ValueError(msg)
    if status == TOEP_ERR_SINGULAR:
        raise errors.SingularMatrix(msg)
    if status == TOEP_ERR_SINGULAR_BLOCK:
        raise errors.SingularBlock(msg)
    if status == TOEP_ERR_SINGULAR_DENOM:
        raise errors.SingularDenominator(-1, msg)
    if status == TOEP_ERR_OOM:
        raise MemoryError(msg)
    raise errors.CudaError(f"libtoepcuda status {status}: {msg}")
