"""Where does the cfg2 operator set-up time go (host generator -> resident spectral blocks)?"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, precompute_spectral  # noqa

torch.cuda.init()
torch.zeros(1, device="cuda")
t0 = time.perf_counter(); s4 = seeded_stacked4(30, 30, 128, 0); t1 = time.perf_counter()
print(f"host generator (RNG) {t1 - t0:.3f} s")
gen = generator_from_stacked(s4); t2 = time.perf_counter(); print(f"generator_from_stacked {t2 - t1:.3f} s")
for i in range(3):
    torch.cuda.synchronize(); t3 = time.perf_counter()
    op = precompute_spectral(gen); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"precompute_spectral #{i} {t4 - t3:.3f} s")
    del op
pinned = torch.from_numpy(s4).pin_memory()
g2 = generator_from_stacked(pinned.numpy())
for i in range(2):
    torch.cuda.synchronize(); t3 = time.perf_counter()
    op = precompute_spectral(g2); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"precompute_spectral from pinned #{i} {t4 - t3:.3f} s")
