"""Debug: device matvec vs the oracle for one (ny, nx, nb, w)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import mlfft  # noqa
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, precompute_spectral  # noqa

ny, nx, nb, w, seed = [int(v) for v in sys.argv[1:6]]
s4 = seeded_stacked4(ny, nx, nb, seed=seed)
gen = generator_from_stacked(s4)
op = precompute_spectral(gen)
u = dense_rhs(gen.dim, w, seed=10)
got = matvec(op, torch.from_numpy(u).cuda()).cpu().numpy()
ref = mlfft.matvec(mlfft.precompute_spectral(s4), (ny, nx, nb, 2 * ny - 1, 2 * nx - 1), u)
print("rel err vs oracle", np.linalg.norm(got - ref) / np.linalg.norm(ref))
