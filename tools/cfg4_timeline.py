"""GPU timeline of a cfg4 GMRES solve (CUPTI): per-step kernel starts/ends."""
import os, sys
import torch
from torch.profiler import ProfilerActivity, profile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, solve_multi_rhs_vectorized  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked  # noqa

sys_ = system_from_generator(generator_from_stacked(seeded_stacked4(64, 64, 128, 0)))
op = BorderedOperator.from_system(sys_)
b = torch.from_numpy(unit_feed_rhs(64, 64, 128)[:, None]).cuda()
for _ in range(2):
    solve_multi_rhs_vectorized(op, None, b, GmresConfig(tol=1e-6, restart=50))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    x, rep = solve_multi_rhs_vectorized(op, None, b, GmresConfig(tol=1e-6, restart=50))
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
print("iterations", rep.iterations, "span", ev[-1].time_range.end - t0)
for e in ev[60:80]:
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f}  {e.name[:60]}")
