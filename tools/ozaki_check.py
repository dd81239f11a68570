"""Multi-RHS matvec: Ozaki (int8 tensor cores) vs the 3M DMMA path vs the oracle; timing."""
import os, subprocess, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4, unit_feed_rhs  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, precompute_spectral  # noqa

ny, nx, nb, w = [int(v) for v in sys.argv[1:5]]
gen = generator_from_stacked(seeded_stacked4(ny, nx, nb, seed=0))
op = precompute_spectral(gen)
u = torch.from_numpy(dense_rhs(gen.dim, w, seed=3)).cuda()
for _ in range(2):
    v = matvec(op, u)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); v = matvec(op, u); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
out = v.cpu().numpy()
tag = os.environ.get("TOEP_MRHS_OZAKI", "1")
np.save(f"/tmp/mv_{tag}.npy", out)
print("ozaki" if tag == "1" else "3M", "ms", sorted(ts)[2], flush=True)
if tag == "1" and os.path.exists("/tmp/mv_0.npy"):
    ref = np.load("/tmp/mv_0.npy")
    print("rel diff vs 3M", np.linalg.norm(out - ref) / np.linalg.norm(ref),
          "max col rel", float(np.max(np.linalg.norm(out - ref, axis=0) / np.linalg.norm(ref, axis=0))))
