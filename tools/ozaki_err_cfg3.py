"""Accuracy of the int8 tensor-core (Ozaki) per-bin products at cfg3's own shape (60x60 grid,
N_b = 256, W = 32): relative error per column against the single-column FP64 path, and column 0
against the reference's cfg3 matvec output (tests/golden/cfg3.npz)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, precompute_spectral  # noqa

op = precompute_spectral(generator_from_stacked(seeded_stacked4(30, 30, 256, seed=0)))
n = 30 * 30 * 256
u = torch.from_numpy(dense_rhs(n, 32, seed=7)).cuda()
u[:, 0] = torch.from_numpy(dense_rhs(n, seed=1)).cuda()
v = matvec(op, u).cpu().numpy()
errs = []
for c in range(32):
    s = matvec(op, u[:, c].contiguous()).cpu().numpy()
    errs.append(float(np.linalg.norm(v[:, c] - s) / np.linalg.norm(s)))
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "cfg3.npz"))
e_ref = float(np.linalg.norm(v[::97, 0] - g["mv_sub"]) / np.linalg.norm(g["mv_sub"]))
e_ref_single = float(np.linalg.norm(matvec(op, u[:, 0].contiguous()).cpu().numpy()[::97] - g["mv_sub"]) /
                     np.linalg.norm(g["mv_sub"]))
out = {"shape": "cfg3 60x60 grid, N_b=256, W=32", "int8_vs_fp64_single_column_rel_err_max": max(errs),
       "int8_vs_fp64_single_column_rel_err_median": float(np.median(errs)),
       "int8_col0_vs_reference_rel_err": e_ref, "fp64_single_col0_vs_reference_rel_err": e_ref_single}
print(json.dumps(out))
