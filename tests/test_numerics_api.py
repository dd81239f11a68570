"""Block-arithmetic helpers and the dense assembly of the reference API surface.

Host paths (numpy in, numpy out) follow the reference's numerics.py:99-123 and problems.py:200-205;
the CUDA-tensor path of ``matmul`` goes through the library's hand-written GEMM (``toep_gemm``).
"""
import numpy as np
import pytest

from paper_2506_20350_b200 import numerics as nm
from paper_2506_20350_b200.errors import DimensionMismatch, ShapeError, TooLargeForOracle
from paper_2506_20350_b200.problems import (BorderedSystem, assemble_full, seeded_stacked4,
                                            system_from_generator)
from paper_2506_20350_b200.toeplitz import assemble_dense, generator_from_stacked


def _rand(shape, seed):
    r = np.random.default_rng(seed)
    return r.standard_normal(shape) + 1j * r.standard_normal(shape)


def test_matmul_host_contract():
    a, b, c = _rand((5, 7), 0), _rand((7, 3), 1), _rand((5, 3), 2)
    np.testing.assert_allclose(nm.matmul(a, b), a @ b, rtol=0, atol=1e-14)
    np.testing.assert_allclose(nm.matmul(a, b, accumulate=c, sign=-1), c - a @ b, rtol=0, atol=1e-14)
    with pytest.raises(DimensionMismatch):
        nm.matmul(a, b.T)
    with pytest.raises(DimensionMismatch):
        nm.matmul(a, b, accumulate=c.T)
    with pytest.raises(ValueError):
        nm.matmul(a, b, sign=2)
    with pytest.raises(ShapeError):
        nm.matmul(a[0], b)


def test_norms():
    a = _rand((4, 6), 3)
    n = nm.norms(a)
    assert n.frobenius == pytest.approx(np.linalg.norm(a)) and n.max_abs == pytest.approx(np.abs(a).max())
    assert nm.norms(np.zeros((0, 3))) == nm.Norms(0.0, 0.0)


def test_assemble_full_blocks_and_cap():
    gen = generator_from_stacked(seeded_stacked4(3, 2, 4, 0))
    s0 = system_from_generator(gen)
    np.testing.assert_array_equal(assemble_full(s0), assemble_dense(gen))
    zb, zc = _rand((2, gen.dim), 4), _rand((2, 2), 5)
    full = assemble_full(BorderedSystem(gen, zb, zc))
    n = gen.dim
    assert full.shape == (n + 2, n + 2)
    np.testing.assert_array_equal(full[:n, :n], assemble_dense(gen))
    np.testing.assert_array_equal(full[:n, n:], zb.T)  # plain transpose, as the reference
    np.testing.assert_array_equal(full[n:, :n], zb)
    np.testing.assert_array_equal(full[n:, n:], zc)
    with pytest.raises(TooLargeForOracle):
        assemble_full(s0, cap=gen.dim - 1)


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k", [(64, 64, 64), (130, 37, 257), (1, 5, 3)])
def test_matmul_device_matches_host(m, n, k):
    import torch

    a, b, c = _rand((m, k), 6), _rand((k, n), 7), _rand((m, n), 8)
    ta, tb, tc = (torch.from_numpy(x).cuda() for x in (a, b, c))
    scale = np.abs(a).sum(axis=1).max() * np.abs(b).max()
    out = nm.matmul(ta, tb)
    assert out.is_cuda
    np.testing.assert_allclose(out.cpu().numpy(), a @ b, rtol=0, atol=1e-13 * scale)
    out = nm.matmul(ta, tb.T.contiguous().T, accumulate=tc, sign=-1)  # column-major operand
    np.testing.assert_allclose(out.cpu().numpy(), c - a @ b, rtol=0, atol=1e-13 * scale)
    np.testing.assert_array_equal(tc.cpu().numpy(), c)  # the accumulator is not modified
    n2 = nm.norms(ta)
    assert n2.frobenius == pytest.approx(np.linalg.norm(a)) and n2.max_abs == pytest.approx(np.abs(a).max())
    with pytest.raises(DimensionMismatch):
        nm.matmul(ta, torch.zeros((k + 1, n), dtype=torch.complex128, device="cuda"))


def test_block_inverse_and_lu_contract():
    a = _rand((9, 9), 11) + 9 * np.eye(9)
    f = nm.lu_factor(a)
    np.testing.assert_allclose(nm.block_inverse(f) @ a, np.eye(9), rtol=0, atol=1e-13)
    b = _rand((9, 3), 12)
    np.testing.assert_allclose(a @ nm.lu_solve(f, b), b, rtol=0, atol=1e-12)
    np.testing.assert_allclose(a.conj().T @ nm.lu_solve(f, b, adjoint=True), b, rtol=0, atol=1e-12)
    with pytest.raises(DimensionMismatch):
        nm.lu_solve(f, b[:-1])


def test_baseline_configs_table_matches_baseline_json():
    import json
    import os
    import re

    from paper_2506_20350_b200.problems import CONFIGS

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "BASELINE.json")
    if not os.path.exists(path):
        pytest.skip("BASELINE.json not shipped")
    texts = json.load(open(path))["configs"]
    assert len(texts) == len(CONFIGS) == 5
    for spec, text in zip(CONFIGS.values(), texts):
        grid = re.search(r"(\d+)\s*[×x]\s*(\d+)", text)
        nb = re.search(r"N_b\s*=\s*(\d+)", text)
        assert (int(grid.group(1)), int(grid.group(2)), int(nb.group(1))) == (spec.ny, spec.nx, spec.nb), text
        assert spec.dim == spec.ny * spec.nx * spec.nb
