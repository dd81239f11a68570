"""Ordered kernel list (start, end, duration) of one cfg3 multi-RHS matvec (CUPTI via torch.profiler).
PDL-launched kernels start before their predecessor ends, so the critical path is read from the
start/end columns, not from the summed durations."""
import os, sys
import torch
from torch.profiler import ProfilerActivity, profile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec  # noqa

op = BorderedOperator.from_system(system_from_generator(generator_from_stacked(seeded_stacked4(30, 30, 256, 0))))
B = torch.from_numpy(unit_feed_rhs(30, 30, 256, columns="each")).cuda()
for _ in range(2):
    matvec(op.spectral, B)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    matvec(op.spectral, B)
    torch.cuda.synchronize()
ev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA), key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = t0
for e in ev:
    s, t = e.time_range.start - t0, e.time_range.end - t0
    print(f"{s:9.1f} {t:9.1f} {t - s:8.1f}  excl {t - max(s, prev_end):8.1f}  {e.name[:90]}")
    prev_end = max(prev_end, t)
print("span us", ev[-1].time_range.end - t0)
