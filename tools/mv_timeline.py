"""GPU timeline of back-to-back cfg2 matvecs (CUPTI): kernel start/end (PDL-launched kernels start early)."""
import os, sys
import torch
from torch.profiler import ProfilerActivity, profile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4, system_from_generator  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec  # noqa

op = BorderedOperator.from_system(system_from_generator(generator_from_stacked(seeded_stacked4(30, 30, 128, 0))))
u = torch.from_numpy(dense_rhs(op.dim, seed=1)[:, None]).cuda()
for _ in range(20):
    matvec(op.spectral, u)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(6):
        matvec(op.spectral, u)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev[3:15]:
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f}  {e.name[:60]}")
