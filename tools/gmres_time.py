"""cfg2 GMRES(50) to 1e-8 solve times (none / PK): median of 9 CUDA-event-timed solves after 2 warm-ups."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, build_pk, solve_multi_rhs_vectorized  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked  # noqa

sys_ = system_from_generator(generator_from_stacked(seeded_stacked4(30, 30, 128, 0)))
op = BorderedOperator.from_system(sys_)
b = torch.from_numpy(unit_feed_rhs(30, 30, 128)[:, None]).cuda()
out = {}
for tag, p in (("none", None), ("pk", build_pk(sys_))):
    for _ in range(2):
        solve_multi_rhs_vectorized(op, p, b, GmresConfig(tol=1e-8, restart=50))
    ts = []
    for _ in range(9):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize()
        e0.record()
        x, rep = solve_multi_rhs_vectorized(op, p, b, GmresConfig(tol=1e-8, restart=50))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out[tag] = {"iterations": rep.iterations, "median_ms": float(np.median(ts)), "min_ms": float(min(ts))}
print(json.dumps(out))
