"""Hand-written FP64 tensor-core GEMMs (csrc/dmma.cu) against an fp64 reference of the same
product: real (toep_dgemm) and complex (toep_gemm) for every operand orientation, ragged sizes
(tile edges in m, n and k), batches with positive and negative batch strides, alpha / beta."""

import ctypes

import numpy as np
import pytest
import torch

from conftest import rel_err
from paper_2506_20350_b200 import _lib

pytestmark = pytest.mark.gpu


def _operand(rows, cols, col_major, batch, dtype, gen, neg=False):
    """(batch, rows, cols) values and a device buffer holding them with the given orientation;
    returns (values, ptr, rs, cs, bs, keepalive)."""
    vals = torch.randn(batch, rows, cols, dtype=dtype, generator=gen)
    if col_major:
        store = vals.transpose(1, 2).contiguous()  # (batch, cols, rows)
        rs, cs = 1, rows
    else:
        store = vals.contiguous()
        rs, cs = cols, 1
    bs = rows * cols
    dev = store.cuda()
    ptr = dev.data_ptr()
    if neg and batch > 1:  # walk the batch backwards: pointer at the last block, negative stride
        ptr += (batch - 1) * bs * dev.element_size()
        bs = -bs
        vals = vals.flip(0)
    return vals, ptr, rs, cs, bs, dev


CASES = [(37, 53, 29, 1), (64, 64, 16, 1), (130, 70, 257, 2), (1, 65, 40, 1), (65, 1, 33, 3), (300, 200, 513, 1)]


@pytest.mark.parametrize("m,n,k,batch", CASES)
@pytest.mark.parametrize("a_cm,b_cm,c_cm", [(0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0), (0, 0, 1), (1, 1, 1)])
def test_dgemm_orientations(m, n, k, batch, a_cm, b_cm, c_cm):
    g = torch.Generator().manual_seed(m * 131 + n * 7 + k + 1000 * a_cm + 100 * b_cm + 10 * c_cm)
    a, ap, ars, acs, abs_, ak = _operand(m, k, a_cm, batch, torch.float64, g, neg=True)
    b, bp, brs, bcs, bbs, bk = _operand(k, n, b_cm, batch, torch.float64, g)
    c, cp, crs, ccs, cbs, ck = _operand(m, n, c_cm, batch, torch.float64, g)
    alpha, beta = 1.25, -0.5
    want = alpha * torch.matmul(a, b) + beta * c
    _lib.check(_lib.lib().toep_dgemm(m, n, k, alpha, ap, ars, acs, abs_, bp, brs, bcs, bbs, beta, cp, crs, ccs, cbs,
                                     batch, _lib.stream_handle()), "dgemm")
    got = ck.cpu()
    if c_cm:
        got = got.transpose(1, 2)
    assert rel_err(got.numpy(), want.numpy()) <= 1e-14


@pytest.mark.parametrize("m,n,k,batch", CASES)
@pytest.mark.parametrize("a_cm,b_cm,c_cm", [(0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0), (0, 0, 1), (1, 0, 1)])
def test_zgemm_orientations(m, n, k, batch, a_cm, b_cm, c_cm):
    g = torch.Generator().manual_seed(m * 31 + n * 17 + k + 1000 * a_cm + 100 * b_cm + 10 * c_cm)
    a, ap, ars, acs, abs_, ak = _operand(m, k, a_cm, batch, torch.complex128, g, neg=True)
    b, bp, brs, bcs, bbs, bk = _operand(k, n, b_cm, batch, torch.complex128, g)
    c, cp, crs, ccs, cbs, ck = _operand(m, n, c_cm, batch, torch.complex128, g)
    alpha, beta = 0.75 - 0.5j, 0.25 + 1.0j
    want = alpha * torch.matmul(a, b) + beta * c
    al = (ctypes.c_double * 2)(alpha.real, alpha.imag)
    be = (ctypes.c_double * 2)(beta.real, beta.imag)
    _lib.check(_lib.lib().toep_gemm(_lib.TOEP_C128, m, n, k, al, ap, ars, acs, abs_, bp, brs, bcs, bbs, be, cp, crs,
                                    ccs, cbs, batch, _lib.stream_handle()), "gemm")
    got = ck.cpu()
    if c_cm:
        got = got.transpose(1, 2)
    assert rel_err(got.numpy(), want.numpy()) <= 1e-14


def test_dgemm_rybicki_block_sum_shape():
    # the deepest block sum of cfg5: 1024 x 1024 output, K = 15 * 1024, all row-major (3M plane)
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(1024, 15 * 1024, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(15 * 1024, 1024, dtype=torch.float64, device="cuda", generator=g)
    c = torch.empty(1024, 1024, dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().toep_dgemm(1024, 1024, 15 * 1024, 1.0, a.data_ptr(), 15 * 1024, 1, 0, b.data_ptr(), 1024,
                                     1, 0, 0.0, c.data_ptr(), 1024, 1, 0, 1, _lib.stream_handle()), "dgemm")
    want = torch.matmul(a, b)
    assert (torch.linalg.norm(c - want) / torch.linalg.norm(want)).item() <= 1e-14
