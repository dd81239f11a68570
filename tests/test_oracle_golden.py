"""Pin the CPU oracle to the reference: every golden fixture was produced by
running the reference toepsolve (tests/golden/make_golden.py)."""

import numpy as np
import pytest

import oracle
from conftest import golden, rel_err
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4, unit_feed_rhs


def _dims(s4, l=None):
    k2, k1, n0, _ = s4.shape
    n2, n1 = (k2 + 1) // 2, (k1 + 1) // 2
    l2, l1 = (k2, k1) if l is None else l
    return (n2, n1, n0, l2, l1)


def test_generator_matches_reference_stream():
    g = golden("small")
    assert np.array_equal(seeded_stacked4(4, 3, 5, seed=3), g["gen_small"])


def test_small_matvec_transpose_and_pk():
    g = golden("small")
    s4 = seeded_stacked4(3, 4, 6, seed=5)
    d = oracle.precompute_spectral(s4)
    dims = _dims(s4)
    assert rel_err(oracle.matvec(d, dims, g["small_u"]), g["small_mv"]) <= 1e-14
    assert rel_err(oracle.matvec_transpose(d, dims, g["small_u"]), g["small_mvt"]) <= 1e-14
    f = oracle.pk_factor(s4[0, 0])
    assert rel_err(oracle.pk_apply(f, g["small_u"]), g["small_pk"]) <= 1e-14


def test_embedding_length_invariance():
    """2n (device) vs 2n-1 (reference) embedding: same matvec."""
    g = golden("small")
    s4 = seeded_stacked4(3, 4, 6, seed=5)
    for l in ((6, 8), (7, 9), (5, 7)):
        d = oracle.precompute_spectral(s4, *l)
        assert rel_err(oracle.matvec(d, _dims(s4, l), g["small_u"]), g["small_mv"]) <= 1e-13


def test_sweep_30_generators():
    g = golden("sweep")
    for i in range(30):
        s4 = g[f"sweep{i}_gen"]
        d = oracle.precompute_spectral(s4)
        got = oracle.matvec(d, _dims(s4), g[f"sweep{i}_u"])
        assert rel_err(got, g[f"sweep{i}_out"]) <= 1e-13
        assert rel_err(got, oracle.assemble_dense(s4) @ g[f"sweep{i}_u"]) <= 1e-12


def test_cfg1_matvec_and_gmres():
    g = golden("cfg1")
    s4 = seeded_stacked4(4, 4, 32, seed=0)
    d = oracle.precompute_spectral(s4)
    dims = _dims(s4)
    assert rel_err(oracle.matvec(d, dims, g["u"]), g["mv"]) <= 1e-14
    b = unit_feed_rhs(4, 4, 32)
    f = oracle.pk_factor(s4[0, 0])
    for tag, prec in (("none", None), ("pk", lambda v: oracle.pk_apply(f, v))):
        x, info = oracle.gmres(lambda v: oracle.matvec(d, dims, v), prec, b, tol=1e-8, restart=30)
        assert info["iterations"] == int(g[f"gm_{tag}_iters"])
        assert np.allclose(info["history"], g[f"gm_{tag}_hist"], rtol=1e-6, atol=1e-14)
        assert rel_err(x, g[f"gm_{tag}_x"]) <= 1e-10


def test_small_rybicki():
    g = golden("small")
    s4 = seeded_stacked4(4, 3, 4, seed=9)
    lvl1 = oracle.assemble_level1(s4)
    x = oracle.rybicki_solve(lvl1, g["ryb_small_y"])
    assert rel_err(x, g["ryb_small_x"]) <= 1e-12


@pytest.mark.slow
def test_cfg2_oracle_matvec_subsample():
    g = golden("cfg2")
    s4 = seeded_stacked4(30, 30, 128, seed=0)
    d = oracle.precompute_spectral(s4)
    mv = oracle.matvec(d, _dims(s4), dense_rhs(30 * 30 * 128, seed=1))
    assert rel_err(mv[::97], g["mv_sub"]) <= 1e-13
