"""Kernel-time breakdown of the cfg3 900-column batched GMRES (CUPTI via torch.profiler)."""
import collections, os, sys
import torch
from torch.profiler import ProfilerActivity, profile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, solve_multi_rhs_sequential  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked  # noqa

sys_ = system_from_generator(generator_from_stacked(seeded_stacked4(30, 30, 256, 0)))
op = BorderedOperator.from_system(sys_)
B = torch.from_numpy(unit_feed_rhs(30, 30, 256, columns="each")).cuda()
solve_multi_rhs_sequential(op, None, B, GmresConfig(tol=1e-6))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    x, reps = solve_multi_rhs_sequential(op, None, B, GmresConfig(tol=1e-6))
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
span = ev[-1].time_range.end - ev[0].time_range.start
tot = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    tot[e.name[:90]][0] += 1
    tot[e.name[:90]][1] += e.time_range.elapsed_us()
print(f"span {span / 1e3:.1f} ms  kernels {len(ev)}")
for k, (c, busy) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:20]:
    print(f"{c:6d}  {busy / 1e3:9.2f} ms  ({busy / c:9.1f} us/launch)  {k}")
# idle gaps between consecutive device activities (host-side stalls show up here)
gaps = []
end = ev[0].time_range.end
for a in ev[1:]:
    g = a.time_range.start - end
    if g > 200:
        gaps.append((g, a.name[:60]))
    end = max(end, a.time_range.end)
print(f"gaps > 0.2 ms: {len(gaps)}, total {sum(g for g, _ in gaps) / 1e3:.1f} ms")
for g, nm in sorted(gaps, reverse=True)[:12]:
    print(f"  {g / 1e3:8.2f} ms before {nm}")
