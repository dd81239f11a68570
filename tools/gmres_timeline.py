"""GPU timeline of one cfg2 GMRES solve (CUPTI via torch.profiler): per-kernel durations and gaps."""
import collections, json, os, sys
import torch
from torch.profiler import ProfilerActivity, profile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, build_pk, solve_multi_rhs_vectorized  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked  # noqa

sys_ = system_from_generator(generator_from_stacked(seeded_stacked4(30, 30, 128, 0)))
op = BorderedOperator.from_system(sys_)
b = torch.from_numpy(unit_feed_rhs(30, 30, 128)[:, None]).cuda()
p = build_pk(sys_) if "pk" in sys.argv[1:] else None
if "notimings" in sys.argv[1:]:
    import importlib; G = importlib.import_module("paper_2506_20350_b200.solvers.gmres")
    _orig = G._run
    G._run = lambda *a, **k: _orig(*a, **{**k, "timings": False})
for _ in range(0 if "fresh" in sys.argv[1:] else 2):  # fresh: profile the first solves (after one plain solve)
    solve_multi_rhs_vectorized(op, p, b, GmresConfig(tol=1e-8, restart=50))
if "fresh" in sys.argv[1:]:
    solve_multi_rhs_vectorized(op, None, b, GmresConfig(tol=1e-8, restart=50))
    if p is not None:
        solve_multi_rhs_vectorized(op, p, b, GmresConfig(tol=1e-8, restart=50))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    x, rep = solve_multi_rhs_vectorized(op, p, b, GmresConfig(tol=1e-8, restart=50))
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
tot = collections.defaultdict(lambda: [0, 0.0, 0.0])  # count, busy, gap-before
prev_end = None
for e in ev:
    name = e.name[:60]
    gap = 0.0 if prev_end is None else max(0.0, e.time_range.start - prev_end)
    tot[name][0] += 1
    tot[name][1] += e.time_range.elapsed_us()
    tot[name][2] += gap
    prev_end = max(prev_end or 0, e.time_range.end)
span = ev[-1].time_range.end - t0
print(f"iterations {rep.iterations}  span {span:.0f} us  kernels {len(ev)}")
for k, (c, busy, gap) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{c:5d}  busy {busy:9.1f} us  ({busy / c:7.1f}/launch)  gaps-before {gap:8.1f} us   {k}")
print("--- timeline: first 14 and last 14 kernels (start, end relative us)")
for e in ev[:14] + ev[-14:]:
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f}  {e.name[:70]}")
