"""Per-call cost split of the host-in / host-out matvec (cfg2): Python allocation of the pinned
output, the single library call with fixed buffers, and the public call."""
import ctypes
import os
import sys
import time

import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200 import _lib  # noqa: E402
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4  # noqa: E402
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, pin, pinned_empty, precompute_spectral  # noqa

op = precompute_spectral(generator_from_stacked(seeded_stacked4(30, 30, 128, 0)))
n = op.dim
uh = pin(dense_rhs(n, seed=1)[:, None])
vh = pinned_empty(uh.shape)
L = _lib.lib()
st = _lib.stream_handle()


def wall(fn, reps=300):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6


print("pinned_empty           us: %.1f" % wall(lambda: pinned_empty(uh.shape)))
print("is_pinned              us: %.1f" % wall(lambda: uh.is_pinned()))
print("stream_handle          us: %.1f" % wall(lambda: _lib.stream_handle()))
print("lib matvec_host        us: %.1f" % wall(lambda: L.toep_matvec_host(op.handle, uh.data_ptr(), vh.data_ptr(), 1, 0, st)))
print("matvec(op, uh)         us: %.1f" % wall(lambda: matvec(op, uh)))
ud = uh.cuda()
print("matvec(op, ud) +sync   us: %.1f" % wall(lambda: (matvec(op, ud), torch.cuda.current_stream().synchronize())))
