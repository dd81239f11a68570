"""cfg2 GMRES(50) solve times, every one of 9 solves per preconditioner, three rounds (spread / outliers)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator, unit_feed_rhs
from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, build_pk, solve_multi_rhs_vectorized
from paper_2506_20350_b200.toeplitz import generator_from_stacked
sys_ = system_from_generator(generator_from_stacked(seeded_stacked4(30, 30, 128, 0)))
op = BorderedOperator.from_system(sys_)
b = torch.from_numpy(unit_feed_rhs(30, 30, 128)[:, None]).cuda()
pk = build_pk(sys_)
for rep in range(3):
    for tag, p in (("none", None), ("pk", pk)):
        for _ in range(2):
            solve_multi_rhs_vectorized(op, p, b, GmresConfig(tol=1e-8, restart=50))
        ts = []
        for _ in range(9):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            torch.cuda.synchronize(); e0.record()
            x, r = solve_multi_rhs_vectorized(op, p, b, GmresConfig(tol=1e-8, restart=50))
            e1.record(); torch.cuda.synchronize(); ts.append(round(e0.elapsed_time(e1), 2))
        print(tag, r.iterations, ts)
