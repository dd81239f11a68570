"""cfg2 host-in / host-out matvec per call (pinned out= path and numpy path): min / median us over
300 calls after 100 warm-up calls, plus the result checked against the device-resident matvec."""
import os
import sys
import time

import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4  # noqa: E402
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, pin, pinned_empty, precompute_spectral  # noqa

op = precompute_spectral(generator_from_stacked(seeded_stacked4(30, 30, 128, 0)))
u_np = dense_rhs(op.dim, seed=1)
uh = pin(u_np[:, None])
vh = pinned_empty(uh.shape, uh.dtype)
ref = matvec(op, torch.from_numpy(u_np[:, None]).cuda()).cpu().numpy()[:, 0]


def percall(fn, reps=300, warm=100):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    ts = np.array(ts) * 1e6
    return ts.min(), np.median(ts)


mn, md = percall(lambda: matvec(op, uh, out=vh))
err = np.linalg.norm(vh.numpy()[:, 0] - ref) / np.linalg.norm(ref)
print(f"pinned out=: min {mn:.1f} us  median {md:.1f} us  ({1e6 / md:.0f} matvec/s)  err {err:.1e}")
r = [None]


def np_call():
    r[0] = matvec(op, u_np)


mn, md = percall(np_call)
err = np.linalg.norm(r[0] - ref) / np.linalg.norm(ref)
print(f"numpy:       min {mn:.1f} us  median {md:.1f} us  ({1e6 / md:.0f} matvec/s)  err {err:.1e}")
