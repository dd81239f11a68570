"""One block-Rybicki solve (N blocks of side s) for launch-list profiling."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.solvers import rybicki_solve  # noqa
N = int(sys.argv[1]) if len(sys.argv) > 1 else 3
s = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
rng = np.random.default_rng(0)
blocks = torch.from_numpy(rng.standard_normal((2 * N - 1, s, s)) + 1j * rng.standard_normal((2 * N - 1, s, s))).cuda()
blocks[0] += 4 * np.sqrt(s) * torch.eye(s, dtype=torch.complex128, device="cuda")
y = torch.from_numpy(rng.standard_normal((N * s, 4)) + 0j).cuda()
x = rybicki_solve(blocks, y)
torch.cuda.synchronize()
print("ok")
