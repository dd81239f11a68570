"""Host-side cost of one cfg2 GMRES call outside the C solve: cProfile of 20 solves, and the
wall time of the Python call against the C library's own t_total."""
import cProfile, os, pstats, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, build_pk, solve_multi_rhs_vectorized  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked  # noqa

sys_ = system_from_generator(generator_from_stacked(seeded_stacked4(30, 30, 128, 0)))
op = BorderedOperator.from_system(sys_)
b = torch.from_numpy(unit_feed_rhs(30, 30, 128)[:, None]).cuda()
for _ in range(3):
    solve_multi_rhs_vectorized(op, None, b, GmresConfig(tol=1e-8, restart=50))
torch.cuda.synchronize()
walls, ctot = [], []
for _ in range(10):
    t0 = time.perf_counter()
    x, rep = solve_multi_rhs_vectorized(op, None, b, GmresConfig(tol=1e-8, restart=50))
    walls.append(time.perf_counter() - t0)
    ctot.append(rep.phase_timings["total"])
print("wall ms", [round(w * 1e3, 3) for w in walls])
print("_run total ms", [round(w * 1e3, 3) for w in ctot])
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    solve_multi_rhs_vectorized(op, None, b, GmresConfig(tol=1e-8, restart=50))
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
