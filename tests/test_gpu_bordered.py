"""Bordered systems (nb > 0) and the PZ row preconditioner.

The reference tests its bordered operator, border LU and Schur step against dense assembly
(test_precond.py / test_rybicki.py pattern); so do these.  GMRES iteration counts are checked
against the oracle's restated MGS-GMRES (oracle/mlfft.py) on the same dense operator, ±1.
"""

import numpy as np
import pytest
import scipy.linalg

from conftest import rel_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import mlfft  # noqa: E402  (test infrastructure: the checker)
from paper_2506_20350_b200.problems import BorderedSystem, seeded_stacked4  # noqa: E402
from paper_2506_20350_b200.solvers import (BorderedOperator, GmresConfig, bordered_matvec, build_pk,  # noqa: E402
                                           build_pz, gmres, schur_solve)
from paper_2506_20350_b200.solvers.bordered import (bordered_matvec_adjoint,  # noqa: E402
                                                    bordered_matvec_transpose)
from paper_2506_20350_b200.toeplitz import (assemble_dense, assemble_dense_1l,  # noqa: E402
                                            generator_from_stacked)

NY, NX, NB, NBORD = 3, 3, 16, 3


def _system(seed=3):
    gen = generator_from_stacked(seeded_stacked4(NY, NX, NB, seed=seed))
    rng = np.random.default_rng(seed + 100)
    n = gen.dim
    zb = (rng.standard_normal((NBORD, n)) + 1j * rng.standard_normal((NBORD, n))) / np.sqrt(n)
    zc = (rng.standard_normal((NBORD, NBORD)) + 1j * rng.standard_normal((NBORD, NBORD))) + 4 * np.eye(NBORD)
    sys_ = BorderedSystem(gen, zb, zc)
    dense = np.block([[assemble_dense(gen), zb.T], [zb, zc]])
    return sys_, dense


def _rand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def test_bordered_matvec_transpose_adjoint_vs_dense():
    sys_, dense = _system()
    op = BorderedOperator.from_system(sys_)
    rng = np.random.default_rng(0)
    x = _rand(rng, sys_.dim, 3)
    assert rel_err(bordered_matvec(op, x), dense @ x) <= 1e-12
    assert rel_err(bordered_matvec_transpose(op, x), dense.T @ x) <= 1e-12
    assert rel_err(bordered_matvec_adjoint(op, x), dense.conj().T @ x) <= 1e-12
    xv = x[:, 0]
    y = bordered_matvec(op, xv)
    assert y.shape == xv.shape and rel_err(y, dense @ xv) <= 1e-12


def test_pk_with_border_lu_vs_dense():
    sys_, dense = _system()
    pk = build_pk(sys_)
    blk = scipy.linalg.block_diag(*([sys_.gen.block(0, 0)] * (NY * NX)), sys_.zc)
    rng = np.random.default_rng(1)
    x = _rand(rng, sys_.dim, 2)
    assert rel_err(pk.apply(x), np.linalg.solve(blk, x)) <= 1e-12
    assert rel_err(pk.apply_adjoint(x), np.linalg.solve(blk.conj().T, x)) <= 1e-12


@pytest.mark.parametrize("bordered", [False, True])
def test_pz_row_preconditioner_vs_dense(bordered):
    sys_, _ = _system()
    if not bordered:
        sys_ = BorderedSystem(sys_.gen, np.zeros((0, sys_.gen.dim), np.complex128), np.zeros((0, 0), np.complex128))
    pz = build_pz(sys_)
    row = assemble_dense_1l(sys_.gen.column(0))
    blocks = [row] * NY + ([sys_.zc] if bordered else [])
    blk = scipy.linalg.block_diag(*blocks)
    rng = np.random.default_rng(2)
    x = _rand(rng, sys_.dim, 2)
    assert rel_err(pz.apply(x), np.linalg.solve(blk, x)) <= 1e-12
    assert rel_err(pz.apply_adjoint(x), np.linalg.solve(blk.conj().T, x)) <= 1e-12


@pytest.mark.parametrize("which", ["pk", "pz"])
def test_gmres_bordered_vs_oracle(which):
    sys_, dense = _system()
    op = BorderedOperator.from_system(sys_)
    p = build_pk(sys_) if which == "pk" else build_pz(sys_)
    rng = np.random.default_rng(4)
    b = _rand(rng, sys_.dim)
    cfg = GmresConfig(tol=1e-10, restart=30)
    x, rep = gmres(lambda v: bordered_matvec(op, v), p, b, cfg)
    assert rep.converged
    assert rel_err(dense @ x, b) <= 1e-9
    pd = np.asarray(p.apply(np.eye(sys_.dim, dtype=np.complex128)))
    _, info = mlfft.gmres(lambda v: dense @ v, lambda v: pd @ v, b, tol=1e-10, restart=30)
    assert abs(rep.iterations - info["iterations"]) <= 1


@pytest.mark.parametrize("inner", ["rybicki", "dense"])
def test_schur_solve_with_border_vs_dense(inner):
    sys_, dense = _system()
    rng = np.random.default_rng(5)
    v = _rand(rng, sys_.dim, 2)
    x, rep = schur_solve(sys_, v, inner)
    assert rep.method == f"schur-{inner}"
    assert rel_err(x, np.linalg.solve(dense, v)) <= 1e-11


def test_tbz1_problem_file_to_device():
    # a bordered problem written by the reference (tests/golden/small.tbz) -> device operator
    import os

    from paper_2506_20350_b200 import problems

    sys_ = problems.load(os.path.join(os.path.dirname(__file__), "golden", "small.tbz"))
    op = BorderedOperator.from_system(sys_)
    dense = np.block([[assemble_dense(sys_.gen), sys_.zb.T], [sys_.zb, sys_.zc]])
    rng = np.random.default_rng(9)
    x = _rand(rng, sys_.dim, 2)
    assert rel_err(bordered_matvec(op, x), dense @ x) <= 1e-12
    v = _rand(rng, sys_.dim, 1)
    sol, _ = schur_solve(sys_, v, "rybicki")
    assert rel_err(sol, np.linalg.solve(dense, v)) <= 1e-10
