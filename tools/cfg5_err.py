"""cfg5 Rybicki solve: error against the reference run's fixture (tests/golden/cfg5.npz) and the
solve time (median of 5 after one warm solve, CUDA events)."""
import os
import sys

import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4, system_from_generator  # noqa: E402
from paper_2506_20350_b200.solvers import schur_solve  # noqa: E402
from paper_2506_20350_b200.toeplitz import generator_from_stacked  # noqa: E402

g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "cfg5.npz"))
gen = generator_from_stacked(seeded_stacked4(16, 16, 64, seed=0))
sys_ = system_from_generator(gen)
y = dense_rhs(gen.dim, 4, seed=1)
x, rep = schur_solve(sys_, y, "rybicki")
xs = x.reshape(-1)[::97]
err = np.linalg.norm(xs - g["x_sub"]) / np.linalg.norm(g["x_sub"])
nerr = abs(np.linalg.norm(x) - g["x_norm"]) / g["x_norm"]
yt = torch.from_numpy(y).cuda()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    e0.record()
    schur_solve(sys_, yt, "rybicki")
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"cfg5: x_sub rel err {err:.2e}, norm rel err {nerr:.2e}, solve {np.median(ts):.1f} ms (min {min(ts):.1f})")
