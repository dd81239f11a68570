"""Per-call host-path matvec latency variants at cfg2 (what makes the pinned path slower than numpy?)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200 import _lib  # noqa
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, pin, pinned_empty, precompute_spectral  # noqa

op = precompute_spectral(generator_from_stacked(seeded_stacked4(30, 30, 128, 0)))
n = op.dim
u_host = pin(dense_rhs(n, seed=1)[:, None])
out = pinned_empty(u_host.shape, u_host.dtype)
out2 = pinned_empty(u_host.shape, u_host.dtype)
u_np = dense_rhs(n, seed=1)
u_pin_np = u_host.numpy()[:, 0].copy()
lib = _lib.lib()
h = op.handle
sh = _lib.stream_handle()
flip = [0]


def raw_pinned():
    _lib.check(lib.toep_matvec_host(h, u_host.data_ptr(), out.data_ptr(), 1, 0, sh))


def raw_pinned_alt():
    flip[0] ^= 1
    _lib.check(lib.toep_matvec_host(h, u_host.data_ptr(), (out if flip[0] else out2).data_ptr(), 1, 0, sh))


def raw_staged():
    _lib.check(lib.toep_matvec_host(h, u_np.__array_interface__["data"][0], out.data_ptr(), 1, 4, sh))


variants = [("api pinned out=", lambda: matvec(op, u_host, out=out)),
            ("api pinned fresh out", lambda: matvec(op, u_host)),
            ("api numpy", lambda: matvec(op, u_np)),
            ("raw ctypes pinned", raw_pinned),
            ("raw ctypes pinned, 2 outs", raw_pinned_alt),
            ("raw ctypes staged numpy", raw_staged)]
for rep in range(2):
    for name, call in variants:
        for _ in range(20):
            call()
        ts = []
        for _ in range(200):
            t0 = time.perf_counter(); call(); ts.append((time.perf_counter() - t0) * 1e6)
        print(f"{name:28s} min {min(ts):6.0f} median {np.median(ts):6.0f} p90 {np.percentile(ts, 90):6.0f} us", flush=True)
