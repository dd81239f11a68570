"""When does the host-path call time settle?  Mean per-call time of the pinned out= matvec in
buckets of 100 calls from the first call of the process; with argument 'spin', the CPU is kept busy
for 1 s (no GPU work) before the first call."""
import os
import sys
import time

import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4  # noqa: E402
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, pin, pinned_empty, precompute_spectral  # noqa

op = precompute_spectral(generator_from_stacked(seeded_stacked4(30, 30, 128, 0)))
uh = pin(dense_rhs(op.dim, seed=1)[:, None])
vh = pinned_empty(uh.shape, uh.dtype)
if "spin" in sys.argv[1:]:
    t_end = time.perf_counter() + 1.0
    x = 0
    while time.perf_counter() < t_end:
        x += 1
ts = np.empty(4000)
for i in range(ts.size):
    t0 = time.perf_counter()
    matvec(op, uh, out=vh)
    ts[i] = time.perf_counter() - t0
b = ts.reshape(-1, 100).mean(axis=1) * 1e6
print(" ".join(f"{v:.0f}" for v in b))
