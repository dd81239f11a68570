"""Phase timestamps of the fused cfg2 matvec (probe library: TOEPCUDA_LIB=.../build_probe/libtoepcuda_probe.so)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, precompute_spectral  # noqa
op = precompute_spectral(generator_from_stacked(seeded_stacked4(30, 30, 128, 0)))
u = torch.from_numpy(dense_rhs(op.dim, seed=1)[:, None]).cuda()
for _ in range(420):
    v = matvec(op, u)
torch.cuda.synchronize()
