"""Matvec time over the first passes of a freshly built operator: the original (precompute_spectral)
and the PK-folded copy (fold_left), in batches of 10 matvecs (CUDA events)."""
import os
import sys

import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4, system_from_generator  # noqa: E402
from paper_2506_20350_b200.solvers import build_pk  # noqa: E402
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, precompute_spectral  # noqa: E402

gen = generator_from_stacked(seeded_stacked4(30, 30, 128, 0))
u = torch.from_numpy(dense_rhs(gen.dim, seed=1)[:, None]).cuda()


def batches(op, tag, n=12):
    out = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10):
            matvec(op, u)
        e1.record()
        torch.cuda.synchronize()
        out.append(round(e0.elapsed_time(e1) * 100, 1))  # us per matvec
    print(tag, out)


op = precompute_spectral(gen)
batches(op, "fresh original")
pk = build_pk(system_from_generator(gen))
folded = op.fold_left(pk.device_blocks()["pinv"])
torch.cuda.synchronize()
batches(folded, "fresh folded  ")
batches(op, "original again")
batches(folded, "folded again  ")
