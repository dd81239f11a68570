import sys; sys.path.insert(0, '.')
import numpy as np, oracle
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, precompute_spectral
for (ny, nx, nb), w in [((16, 16, 64), 70), ((16, 16, 128), 64)]:
    s4 = seeded_stacked4(ny, nx, nb, seed=w); gen = generator_from_stacked(s4); op = precompute_spectral(gen)
    u = dense_rhs(gen.dim, w, seed=5)
    want = oracle.mlfft.matvec(oracle.mlfft.precompute_spectral(s4), (ny, nx, nb, 2*ny-1, 2*nx-1), u)
    got = np.asarray(matvec(op, u))
    print(ny, nx, nb, w, "rel err vs oracle", np.linalg.norm(got - want) / np.linalg.norm(want))
