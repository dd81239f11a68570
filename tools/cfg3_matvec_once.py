"""One cfg3 multi-RHS (W = 900) matvec for kernel profiling (tensor-core per-bin GEMM)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec  # noqa

op = BorderedOperator.from_system(system_from_generator(generator_from_stacked(seeded_stacked4(30, 30, 256, 0))))
B = torch.from_numpy(unit_feed_rhs(30, 30, 256, columns="each")).cuda()
for _ in range(2):
    matvec(op.spectral, B)
torch.cuda.synchronize()
print("ok")
if os.environ.get("NCU_RANGE"):  # ncu --profile-from-start off: capture one steady-state matvec only
    torch.cuda.profiler.start()
    matvec(op.spectral, B)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
