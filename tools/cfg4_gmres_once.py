"""One cfg4 GMRES(50) solve to 1e-6 (dtype from argv: c64 | c128) for kernel launch lists."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, solve_multi_rhs_vectorized  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked  # noqa

dt = torch.complex64 if "c64" in sys.argv[1:] else torch.complex128
sys_ = system_from_generator(generator_from_stacked(seeded_stacked4(64, 64, 128, 0)))
op = BorderedOperator.from_system(sys_, dtype=dt)
b = torch.from_numpy(unit_feed_rhs(64, 64, 128)[:, None]).cuda()
x, rep = solve_multi_rhs_vectorized(op, None, b, GmresConfig(tol=1e-6, restart=50))
torch.cuda.synchronize()
print("iterations", rep.iterations)
