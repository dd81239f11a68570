"""Device LU (toep_lu_factor / toep_lu_solve) against LAPACK zgetrf / zgetrs.

The reference factors every denominator with scipy.linalg.lu_factor (numerics.py:44-66, LAPACK
zgetrf: partial pivoting on |re| + |im|).  The device factorisation uses the same pivot measure,
so for matrices without near-ties the pivot sequence is identical and the factors agree to
rounding; solves agree with LAPACK's to ~1e-12 relative.
"""

import numpy as np
import pytest
import scipy.linalg

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _factor(a_np):
    from paper_2506_20350_b200 import _lib

    n = a_np.shape[0]
    lu = torch.from_numpy(np.ascontiguousarray(a_np)).cuda()
    piv = torch.empty(n, dtype=torch.int32, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().toep_lu_factor(lu.data_ptr(), n, piv.data_ptr(), info.data_ptr(), _lib.stream_handle()),
               "lu_factor")
    torch.cuda.synchronize()
    return lu, piv, int(info.item())


def _solve(lu, piv, b_np):
    from paper_2506_20350_b200 import _lib

    n = lu.shape[0]
    x = torch.from_numpy(np.ascontiguousarray(b_np)).cuda()
    _lib.check(_lib.lib().toep_lu_solve(lu.data_ptr(), n, piv.data_ptr(), x.data_ptr(), x.shape[1],
                                        _lib.stream_handle()), "lu_solve")
    torch.cuda.synchronize()
    return x.cpu().numpy()


def _rand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


@pytest.mark.parametrize("n", [1, 2, 5, 31, 32, 33, 63, 64, 65, 100, 257, 512, 1024, 1500, 2100, 3000])
def test_factor_matches_lapack(n):
    rng = np.random.default_rng(n)
    a = _rand(rng, n, n)
    lu, piv, info = _factor(a)
    assert info == 0
    lu_ref, piv_ref = scipy.linalg.lu_factor(a)
    np.testing.assert_array_equal(piv.cpu().numpy(), piv_ref)
    err = np.linalg.norm(lu.cpu().numpy() - lu_ref) / np.linalg.norm(lu_ref)
    assert err < 1e-12, err


@pytest.mark.parametrize("n,nrhs", [(1, 1), (7, 3), (33, 1), (128, 130), (1024, 4), (1024, 1024)])
def test_solve_matches_lapack(n, nrhs):
    rng = np.random.default_rng(1000 + n)
    a = _rand(rng, n, n)
    b = _rand(rng, n, nrhs)
    lu, piv, _ = _factor(a)
    x = _solve(lu, piv, b)
    x_ref = scipy.linalg.lu_solve(scipy.linalg.lu_factor(a), b)
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) < 1e-11


def test_pivoting_is_exercised():
    # a permuted, strongly graded matrix: every column needs an interchange
    rng = np.random.default_rng(7)
    n = 96
    a = np.diag(np.logspace(0, 6, n)).astype(np.complex128)[rng.permutation(n)] + 1e-3 * _rand(rng, n, n)
    lu, piv, info = _factor(a)
    assert info == 0
    lu_ref, piv_ref = scipy.linalg.lu_factor(a)
    np.testing.assert_array_equal(piv.cpu().numpy(), piv_ref)
    assert (piv_ref != np.arange(n)).sum() > n // 2
    b = _rand(rng, n, 2)
    x = _solve(lu, piv, b)
    assert np.linalg.norm(a @ x - b) / np.linalg.norm(b) < 1e-12


@pytest.mark.parametrize("zero_col", [0, 5, 40])
def test_singular_reports_first_zero_pivot(zero_col):
    rng = np.random.default_rng(3)
    n = 48
    a = _rand(rng, n, n)
    a[:, zero_col] = 0.0
    _, _, info = _factor(a)
    # LAPACK: info = first (1-based) column whose pivot is exactly zero
    _, _, info_ref = scipy.linalg.lapack.zgetrf(a)
    assert info == info_ref == zero_col + 1


def test_too_large_is_an_argument_error():
    from paper_2506_20350_b200 import _lib
    from paper_2506_20350_b200.errors import ToepsolveError

    n = 5000  # > kCL * 2 * 256 rows: beyond the cluster-resident panel (checked before any access)
    lu = torch.empty((1, 1), dtype=torch.complex128, device="cuda")
    piv = torch.empty(1, dtype=torch.int32, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    with pytest.raises((ToepsolveError, ValueError, RuntimeError)):
        _lib.check(_lib.lib().toep_lu_factor(lu.data_ptr(), n, piv.data_ptr(), info.data_ptr(),
                                             _lib.stream_handle()), "lu_factor")
