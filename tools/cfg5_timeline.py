"""CUPTI timeline of one cfg5 Rybicki solve: busy time per stream, per kernel family, and the span."""
import collections
import re
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4, system_from_generator  # noqa: E402
from paper_2506_20350_b200.solvers import schur_solve  # noqa: E402
from paper_2506_20350_b200.toeplitz import generator_from_stacked  # noqa: E402

gen = generator_from_stacked(seeded_stacked4(16, 16, 64, 0))
sys_ = system_from_generator(gen)
y = torch.from_numpy(dense_rhs(gen.dim, 4, seed=1)).cuda()
schur_solve(sys_, y, "rybicki")
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    schur_solve(sys_, y, "rybicki")
    torch.cuda.synchronize()
ev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
            key=lambda e: e.time_range.start)
t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
by_k = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    k = re.sub(r"\(anonymous namespace\)::", "", e.name)
    k = re.split(r"[<(]", k.replace("void ", "").replace("toep::", ""))[0][:60]
    by_k[k][0] += 1
    by_k[k][1] += e.time_range.elapsed_us()
print(f"span {(t1 - t0) / 1e3:.1f} ms, {len(ev)} kernels/copies")
for k, (c, us) in sorted(by_k.items(), key=lambda kv: -kv[1][1])[:14]:
    print(f"{c:5d} {us / 1e3:8.2f} ms  {k}")
# busy union over time (any kernel running)
iv = sorted((e.time_range.start, e.time_range.end) for e in ev)
busy, cur_s, cur_e = 0.0, None, None
for s_, e_ in iv:
    if cur_e is None or s_ > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s_, e_
    else:
        cur_e = max(cur_e, e_)
busy += cur_e - cur_s
print(f"device busy (union) {busy / 1e3:.1f} ms, idle {(t1 - t0 - busy) / 1e3:.1f} ms")

if len(sys.argv) > 1:  # dump (start, end, stream, name) rows for offline analysis
    with open(sys.argv[1], "w") as f:
        for e in ev:
            k = re.sub(r"\(anonymous namespace\)::", "", e.name)
            k = re.split(r"[<(]", k.replace("void ", "").replace("toep::", ""))[0][:40]
            f.write(f"{(e.time_range.start - t0):.1f} {(e.time_range.end - t0):.1f} {getattr(e, 'device_resource_id', -1)} {k}\n")
