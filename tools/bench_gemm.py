"""GEMM throughput: DMMA tensor-core ZGEMM vs SIMT fallback (TOEP_ZGEMM=simt) vs cuBLAS (torch)."""
import ctypes, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200 import _lib  # noqa
lib = _lib.load()
one = (ctypes.c_double * 2)(1.0, 0.0)
zero = (ctypes.c_double * 2)(0.0, 0.0)

def run(name, m, n, k, batch, a, ars, acs, abs_, b, brs, bcs, bbs, c, crs, ccs, cbs, reps=5):
    def go():
        _lib.check(lib.toep_gemm(0, m, n, k, one, a.data_ptr(), ars, acs, abs_, b.data_ptr(), brs, bcs, bbs, zero,
                                 c.data_ptr(), crs, ccs, cbs, batch, _lib.stream_handle()))
    go(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        go()
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    print(f"{name}: {t*1e3:.2f} ms  {8*m*n*k*batch/t/1e12:.2f} TFLOP/s", flush=True)

dev = "cuda"
# cfg3 per-bin: V_k (256x900) = D_k (256x256, col-major) U_k (256x900 row-major), 3600 bins (use 600 to fit fast)
K, n0, W = 600, 256, 900
DT = torch.randn(K, n0, n0, dtype=torch.complex128, device=dev)
U = torch.randn(K, n0, W, dtype=torch.complex128, device=dev)
V = torch.empty(K, n0, W, dtype=torch.complex128, device=dev)
run("per-bin 256x900x256 x600", n0, W, n0, K, DT, 1, n0, n0 * n0, U, W, 1, n0 * W, V, W, 1, n0 * W)
ref = torch.matmul(DT.transpose(1, 2), U)
print("  rel err vs cuBLAS", (torch.linalg.norm(ref - V) / torch.linalg.norm(ref)).item())
t0 = time.time(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record()
for _ in range(5): torch.matmul(DT.transpose(1, 2), U, out=V)
e1.record(); torch.cuda.synchronize(); t = e0.elapsed_time(e1) / 5e3
print(f"  cuBLAS: {t*1e3:.2f} ms {8*n0*W*n0*K/t/1e12:.2f} TFLOP/s")
del DT, U, V, ref
# fold: 128 x 460800 x 128
M = torch.randn(128, 128, dtype=torch.complex128, device=dev)
B = torch.randn(460800, 128, dtype=torch.complex128, device=dev)
C = torch.empty_like(B)
run("fold 128x460800x128", 128, 460800, 128, 1, M, 128, 1, 0, B, 1, 128, 0, C, 1, 128, 0)
ref = B @ M.T
print("  rel err", (torch.linalg.norm(ref - C) / torch.linalg.norm(ref)).item())
del B, C, ref
# rybicki: 1024^3
A = torch.randn(1024, 1024, dtype=torch.complex128, device=dev)
B = torch.randn(1024, 1024, dtype=torch.complex128, device=dev)
C = torch.empty_like(A)
run("dense 1024^3", 1024, 1024, 1024, 1, A, 1024, 1, 0, B, 1024, 1, 0, C, 1024, 1, 0)
ref = A @ B
print("  rel err", (torch.linalg.norm(ref - C) / torch.linalg.norm(ref)).item())
e0.record()
for _ in range(5): torch.matmul(A, B, out=C)
e1.record(); torch.cuda.synchronize(); t = e0.elapsed_time(e1) / 5e3
print(f"  cuBLAS: {t*1e3:.2f} ms {8*1024**3/t/1e12:.2f} TFLOP/s")
