"""Host-side layout logic of the library page-locked tensors (no allocation: runs without a GPU)."""
import numpy as np
import torch

from paper_2506_20350_b200 import hostmem


def test_layout_rounding_and_shapes():
    shp, count, nbytes, btype = hostmem._layout((115200, 1), torch.complex128)
    assert shp == (115200, 1) and count == 115200 and nbytes == 115200 * 16
    assert hostmem._layout(7, torch.complex64)[:3] == ((7,), 7, 4096)
    assert hostmem._layout(np.int64(3), torch.complex128)[:3] == ((3,), 3, 4096)
    assert hostmem._layout(torch.Size([3, 4]), torch.complex128)[:3] == ((3, 4), 12, 4096)
    assert hostmem._layout((), torch.complex128)[:3] == ((), 1, 4096)
    assert hostmem._layout((0, 5), torch.complex128)[1] == 0
    # one ctypes block type per byte size, reused
    assert hostmem._layout((257,), torch.complex128)[3] is hostmem._layout((257, 1), torch.complex128)[3]
