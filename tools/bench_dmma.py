"""Throughput of the hand-written DMMA GEMMs (csrc/dmma.cu) on the shapes the solvers use, next to
cuBLAS (torch.matmul, fp64 / c128) on the same shapes.  FLOP counts: real 2mnk, complex 8mnk."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200 import _lib  # noqa: E402

lib = _lib.load()
dev = "cuda"
res = {}


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def dgemm_case(name, m, n, k, batch=1):
    a = torch.randn(batch, m, k, dtype=torch.float64, device=dev)
    b = torch.randn(batch, k, n, dtype=torch.float64, device=dev)
    c = torch.empty(batch, m, n, dtype=torch.float64, device=dev)

    def ours():
        _lib.check(lib.toep_dgemm(m, n, k, 1.0, a.data_ptr(), k, 1, m * k, b.data_ptr(), n, 1, k * n, 0.0,
                                  c.data_ptr(), n, 1, m * n, batch, _lib.stream_handle()))
    t = timed(ours)
    tc = timed(lambda: torch.matmul(a, b, out=c))
    fl = 2 * m * n * k * batch
    res[name] = {"ours_ms": t * 1e3, "ours_tflops": fl / t / 1e12, "cublas_ms": tc * 1e3, "cublas_tflops": fl / tc / 1e12}
    print(name, json.dumps(res[name]), flush=True)


def zgemm_case(name, m, n, k, batch=1, a_cm=False):
    a = torch.randn(batch, m, k, dtype=torch.complex128, device=dev)
    b = torch.randn(batch, k, n, dtype=torch.complex128, device=dev)
    c = torch.empty(batch, m, n, dtype=torch.complex128, device=dev)
    one = (ctypes.c_double * 2)(1.0, 0.0)
    zero = (ctypes.c_double * 2)(0.0, 0.0)
    at = a.transpose(1, 2).contiguous() if a_cm else a
    ars, acs = (1, m) if a_cm else (k, 1)

    def ours():
        _lib.check(lib.toep_gemm(0, m, n, k, one, at.data_ptr(), ars, acs, m * k, b.data_ptr(), n, 1, k * n, zero,
                                 c.data_ptr(), n, 1, m * n, batch, _lib.stream_handle()))
    t = timed(ours)
    tc = timed(lambda: torch.matmul(a, b, out=c))
    fl = 8 * m * n * k * batch
    res[name] = {"ours_ms": t * 1e3, "ours_tflops": fl / t / 1e12, "cublas_ms": tc * 1e3, "cublas_tflops": fl / tc / 1e12}
    print(name, json.dumps(res[name]), flush=True)


dgemm_case("rybicki_blocksum_1024x1024x15360", 1024, 1024, 15360)
dgemm_case("rybicki_blocksum_1024x1024x4096_b2", 1024, 1024, 4096, 2)
dgemm_case("rybicki_cross_1024x1024x1024_b15", 1024, 1024, 1024, 15)
dgemm_case("dgemm_4096", 4096, 4096, 4096)
dgemm_case("mrhs_3m_plane_256x900x256_b360", 256, 900, 256, 360)
zgemm_case("lu_trailing_992x992x32_b2", 992, 992, 32, 2)
zgemm_case("zgemm_2048", 2048, 2048, 2048)
zgemm_case("perbin_256x900x256_b120_acm", 256, 900, 256, 120, a_cm=True)
zgemm_case("pk_fold_128x460800x128_acm", 128, 460800, 128, 1, a_cm=False)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/bench_dmma.json", "w"), indent=1)
