"""One cfg2 GMRES(50) solve (after a warm-up) for kernel profiling."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, solve_multi_rhs_vectorized  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked  # noqa

sys_ = system_from_generator(generator_from_stacked(seeded_stacked4(30, 30, 128, 0)))
op = BorderedOperator.from_system(sys_)
b = torch.from_numpy(unit_feed_rhs(30, 30, 128)[:, None]).cuda()
for _ in range(2):
    x, rep = solve_multi_rhs_vectorized(op, None, b, GmresConfig(tol=1e-8, restart=50))
torch.cuda.synchronize()
print("ok", rep.iterations)
