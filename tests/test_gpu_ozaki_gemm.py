"""Generic FP64 GEMM on the int8 tensor cores (Ozaki scheme, toep_ozaki_dgemm) against torch's FP64
matmul: the Rybicki block-sum shapes, ragged N, alpha / beta, and a K sub-range of a sliced matrix."""
import numpy as np
import pytest
import torch

from paper_2506_20350_b200 import _lib

pytestmark = pytest.mark.gpu


def ozaki(a, b, c=None, alpha=1.0, beta=0.0):
    m, k = a.shape
    n = b.shape[1]
    out = torch.zeros((m, n), dtype=torch.float64, device="cuda") if c is None else c
    _lib.check(_lib.lib().toep_ozaki_dgemm(m, n, k, alpha, a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), beta,
                                           out.data_ptr(), out.stride(0), _lib.stream_handle()), "ozaki_dgemm")
    return out


@pytest.mark.parametrize("m,n,k", [(128, 128, 32), (256, 100, 512), (1024, 1024, 1024), (1024, 1024, 15360),
                                   (512, 1000, 4096)])
def test_ozaki_dgemm_vs_fp64(m, n, k):
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    a = torch.randn((m, k), dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn((k, n), dtype=torch.float64, device="cuda", generator=g)
    got = ozaki(a, b)
    want = a @ b
    err = (torch.linalg.norm(got - want) / torch.linalg.norm(want)).item()
    assert err <= 3e-13, err  # 7 digits: ~2^-49 per digit product, growing like sqrt(K) on random data


def test_ozaki_dgemm_alpha_beta_and_scaled_rows():
    g = torch.Generator(device="cuda").manual_seed(7)
    a = torch.randn((256, 1024), dtype=torch.float64, device="cuda", generator=g)
    a *= torch.logspace(-6, 6, 256, dtype=torch.float64, device="cuda")[:, None]  # rows over 12 decades
    b = torch.randn((1024, 300), dtype=torch.float64, device="cuda", generator=g)
    c0 = torch.randn((256, 300), dtype=torch.float64, device="cuda", generator=g)
    got = ozaki(a, b, c0.clone(), alpha=-2.0, beta=0.5)
    want = -2.0 * (a @ b) + 0.5 * c0
    rows = torch.linalg.norm(got - want, dim=1) / torch.linalg.norm(want, dim=1)
    assert rows.max().item() <= 1e-13
