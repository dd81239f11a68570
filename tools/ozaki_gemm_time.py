"""Time the generic Ozaki int8 GEMM (toep_ozaki_dgemm, slicing included) against the hand-written
FP64 DMMA GEMM (toep_dgemm) on the Rybicki block-sum shapes."""
import os
import sys

import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200 import _lib  # noqa: E402

L = _lib.lib()
st = _lib.stream_handle()


def t(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for (m, n, k) in [(1024, 1024, 1024), (1024, 1024, 4096), (1024, 1024, 15360)]:
    a = torch.randn((m, k), dtype=torch.float64, device="cuda")
    b = torch.randn((k, n), dtype=torch.float64, device="cuda")
    c = torch.empty((m, n), dtype=torch.float64, device="cuda")
    to = t(lambda: L.toep_ozaki_dgemm(m, n, k, 1.0, a.data_ptr(), k, b.data_ptr(), n, 0.0, c.data_ptr(), n, st))
    td = t(lambda: L.toep_dgemm(m, n, k, 1.0, a.data_ptr(), k, 1, 0, b.data_ptr(), n, 1, 0, 0.0, c.data_ptr(), n, 1, 0,
                                1, st))
    fl = 2.0 * m * n * k
    print(f"{m}x{n}x{k}: ozaki {to:.3f} ms ({fl / to / 1e9:.1f} TFLOP/s)  dmma {td:.3f} ms ({fl / td / 1e9:.1f} TFLOP/s)")
