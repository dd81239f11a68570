"""cfg2 device-resident matvec/s: 1000 back-to-back matvecs after 10 warm-ups, CUDA events."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, precompute_spectral  # noqa
op = precompute_spectral(generator_from_stacked(seeded_stacked4(30, 30, 128, 0)))
u = torch.from_numpy(dense_rhs(op.dim, seed=1)[:, None]).cuda()
for _ in range(10):
    v = matvec(op, u)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(1000):
    v = matvec(op, u)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 1000
print(f"matvec {ms * 1e3:.1f} us  {1.0 / (ms * 1e-3):.0f} matvec/s")
