import os, sys, collections
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator, unit_feed_rhs
from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, solve_multi_rhs_sequential, build_pk
from paper_2506_20350_b200.toeplitz import generator_from_stacked
sys_ = system_from_generator(generator_from_stacked(seeded_stacked4(30, 30, 256, 0)))
op = BorderedOperator.from_system(sys_)
B = torch.from_numpy(unit_feed_rhs(30, 30, 256, columns="each")).cuda()
for tag, p in (("none", None), ("pk", build_pk(sys_))):
    x, reps = solve_multi_rhs_sequential(op, p, B, GmresConfig(tol=1e-6))
    print(tag, sorted(collections.Counter(r.iterations for r in reps).items()))
    h = np.array([r.residual_history[13] if len(r.residual_history) > 13 else 0 for r in reps])
    print(" residual after 13/14 its: max", h.max())
