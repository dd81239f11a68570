"""Distribution of the cfg2 host-in / host-out matvec call time (pinned out= path): percentiles over
2000 calls through the public API, through the bare library call, and with the Python GC off."""
import gc
import os
import sys
import time

import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200 import _lib  # noqa: E402
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4  # noqa: E402
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, pin, pinned_empty, precompute_spectral  # noqa

op = precompute_spectral(generator_from_stacked(seeded_stacked4(30, 30, 128, 0)))
uh = pin(dense_rhs(op.dim, seed=1)[:, None])
vh = pinned_empty(uh.shape, uh.dtype)
L = _lib.lib()
st = _lib.stream_handle()


def dist(tag, fn, n=2000, warm=200):
    for _ in range(warm):
        fn()
    ts = np.empty(n)
    for i in range(n):
        t0 = time.perf_counter()
        fn()
        ts[i] = time.perf_counter() - t0
    ts *= 1e6
    p = np.percentile(ts, [1, 10, 50, 90, 99])
    print(f"{tag:28s} mean {ts.mean():6.1f}  p1 {p[0]:6.1f} p10 {p[1]:6.1f} p50 {p[2]:6.1f} p90 {p[3]:6.1f} "
          f"p99 {p[4]:6.1f} max {ts.max():7.1f} us  -> {1e6 / ts.mean():.0f} matvec/s")


order = sys.argv[1:] or ["public", "bare", "gcoff", "public"]
for o in order:
    if o == "public":
        dist("public matvec(out=)", lambda: matvec(op, uh, out=vh))
    elif o == "bare":
        dist("bare toep_matvec_host", lambda: L.toep_matvec_host(op.handle, uh.data_ptr(), vh.data_ptr(), 1, 0, st))
    elif o == "gcoff":
        gc.disable()
        dist("public, gc off", lambda: matvec(op, uh, out=vh))
        gc.enable()
ud = uh.cuda()
dist("device matvec + sync", lambda: (matvec(op, ud), torch.cuda.current_stream().synchronize()))
