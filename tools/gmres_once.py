"""One cfg2 GMRES(50) solve (for launch-list profiling)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, solve_multi_rhs_vectorized  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked  # noqa
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
sys_ = system_from_generator(generator_from_stacked(seeded_stacked4(n, n, 128, seed=0)))
op = BorderedOperator.from_system(sys_)
b = torch.from_numpy(unit_feed_rhs(n, n, 128)[:, None]).cuda()
x, rep = solve_multi_rhs_vectorized(op, None, b, GmresConfig(tol=1e-8, restart=50))
torch.cuda.synchronize()
print(rep.iterations, rep.final_residual)
