"""The C-ABI library loads on CPU and exports every symbol include/toepcuda.h declares."""

import ctypes
import os
import re

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "toepcuda.h")
LIB = os.path.join(REPO, "paper_2506_20350_b200", "libtoepcuda.so")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"TOEP_API\s+[\w\s\*]*?\b(toep_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("toep_op_create", "toep_matvec", "toep_gmres", "toep_block_apply", "toep_last_error"):
        assert must in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="libtoepcuda.so not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    for name in declared():
        assert hasattr(lib, name), name


@pytest.mark.skipif(not os.path.exists(LIB), reason="libtoepcuda.so not built")
def test_python_binding_covers_header():
    from paper_2506_20350_b200 import _lib

    assert set(_lib.SIGNATURES) == set(declared())
    lib = _lib.load()
    assert lib.toep_version() >= 100
    # error path without a GPU: null arguments are rejected before touching CUDA
    assert lib.toep_matvec(None, None, None, 1, 0, None) == _lib.TOEP_ERR_ARG
    assert "null" in _lib.last_error()
