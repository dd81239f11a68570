"""One cfg5 Rybicki solve (16x16, N_b=64, 4 RHS) for kernel launch lists (after one warm solve)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4, system_from_generator  # noqa
from paper_2506_20350_b200.solvers import schur_solve  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked  # noqa

gen = generator_from_stacked(seeded_stacked4(16, 16, 64, 0))
sys_ = system_from_generator(gen)
y = torch.from_numpy(dense_rhs(gen.dim, 4, seed=1)).cuda()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    x, rep = schur_solve(sys_, y, "rybicki")
torch.cuda.synchronize()
print("ok", rep.phase_timings.get("recursion"))
