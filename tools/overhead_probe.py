import time, torch, sys, os
sys.path.insert(0, '/root/repo')
from paper_2506_20350_b200 import _lib
from paper_2506_20350_b200._tensor import to_columns, restore
n = 115200
uh = torch.randn(n, 1, dtype=torch.complex128).pin_memory()
ud = uh.cuda()
def t(fn, reps=2000):
    for _ in range(50): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6
print("empty pinned", t(lambda: torch.empty((n, 1), dtype=torch.complex128, pin_memory=True)))
print("empty_like dev", t(lambda: torch.empty_like(ud)))
print("stream_handle", t(lambda: _lib.stream_handle()))
print("require_cuda", t(lambda: _lib.require_cuda()))
print("to_columns(dev)", t(lambda: to_columns(ud)))
print("current_stream().synchronize()", t(lambda: torch.cuda.current_stream().synchronize()))
print("raw stream check", _lib.stream_handle() == torch.cuda.current_stream().cuda_stream)
