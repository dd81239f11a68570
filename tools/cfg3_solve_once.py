"""One cfg3 900-column batched GMRES(1e-6) solve (after a warm-up) for kernel profiling."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, solve_multi_rhs_sequential  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked  # noqa

op = BorderedOperator.from_system(system_from_generator(generator_from_stacked(seeded_stacked4(30, 30, 256, 0))))
B = torch.from_numpy(unit_feed_rhs(30, 30, 256, columns="each")).cuda()
solve_multi_rhs_sequential(op, None, B, GmresConfig(tol=1e-6))
torch.cuda.synchronize()
print("warm", flush=True)
torch.cuda.profiler.start()
solve_multi_rhs_sequential(op, None, B, GmresConfig(tol=1e-6))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
