"""TBZ1 problem files (problems.py:219-322 of the reference) — host code, runs without a GPU.

Pinned to a file written by the reference's own ``problems.save`` and the arrays its ``load``
read back (tests/golden/make_golden.py part ``tbz``): our loader must return the same arrays,
our writer must reproduce the reference's bytes exactly, and corrupted / foreign files must raise
the reference's exceptions.
"""

import os

import numpy as np
import pytest

from paper_2506_20350_b200 import problems
from paper_2506_20350_b200.errors import ChecksumMismatch, FormatVersionMismatch, InvalidSpec

HERE = os.path.dirname(os.path.abspath(__file__))
TBZ = os.path.join(HERE, "golden", "small.tbz")


@pytest.fixture(scope="module")
def ref():
    return np.load(os.path.join(HERE, "golden", "tbz.npz"))


def test_load_matches_reference_loader(ref):
    sys_ = problems.load(TBZ)
    np.testing.assert_array_equal(sys_.gen.stacked4(), ref["stacked4"])
    np.testing.assert_array_equal(sys_.zb, ref["zb"])
    np.testing.assert_array_equal(sys_.zc, ref["zc"])
    s = sys_.spec
    assert [s.ny, s.nx, s.ne, s.nb, s.seed] == list(ref["spec"])
    assert [s.wavenumber, s.pitch, s.regularization, s.diagonal_shift] == list(ref["spec_f"])
    assert sys_.dim == s.ny * s.nx * s.ne + s.nb


def test_save_reproduces_reference_bytes(tmp_path):
    sys_ = problems.load(TBZ)
    out = tmp_path / "again.tbz"
    problems.save(sys_, out)
    assert out.read_bytes() == open(TBZ, "rb").read()


def test_fnv1a64_known_answers(ref):
    assert problems.fnv1a64(b"") == 0xCBF29CE484222325
    assert problems.fnv1a64(b"a") == 0xAF63DC4C8601EC8C  # published FNV-1a 64 test vector
    with open(TBZ, "rb") as fh:
        assert problems.fnv1a64(fh.read()[:64]) == int(ref["fnv"][0])


def test_corrupted_payload_and_truncation(tmp_path):
    blob = bytearray(open(TBZ, "rb").read())
    bad = tmp_path / "bad.tbz"
    flipped = bytearray(blob)
    flipped[len(blob) // 2] ^= 0x01
    bad.write_bytes(bytes(flipped))
    with pytest.raises(ChecksumMismatch):
        problems.load(bad)
    bad.write_bytes(bytes(blob[:-9]))
    with pytest.raises(ChecksumMismatch):
        problems.load(bad)
    bad.write_bytes(bytes(blob[:7]))
    with pytest.raises(ChecksumMismatch):
        problems.load(bad)


def test_foreign_magic_and_version(tmp_path):
    blob = open(TBZ, "rb").read()
    bad = tmp_path / "bad.tbz"
    bad.write_bytes(b"TBZ2\n" + blob[5:])
    with pytest.raises(FormatVersionMismatch):
        problems.load(bad)
    hlen = int.from_bytes(blob[5:9], "little")
    header = blob[9:9 + hlen].replace(b'"version": 1', b'"version": 9')
    bad.write_bytes(blob[:9] + header + blob[9 + hlen:])
    with pytest.raises(FormatVersionMismatch):
        problems.load(bad)


def test_spec_validation():
    with pytest.raises(InvalidSpec):
        problems.ArrayProblemSpec(ny=0, nx=1, ne=1)
    with pytest.raises(InvalidSpec):
        problems.ArrayProblemSpec(ny=1, nx=1, ne=1, nb=-1)
    s = problems.ArrayProblemSpec(ny=2, nx=3, ne=4)
    assert s.nb == 8 * (2 + 3) and s.regularization == pytest.approx(0.1)


def test_generate_matches_reference(ref):
    # the golden file was written from the reference's generate() of this spec
    spec = problems.ArrayProblemSpec(ny=2, nx=3, ne=4, nb=5, wavenumber=2.5, pitch=1.0, seed=7)
    sys_ = problems.generate(spec)
    np.testing.assert_allclose(sys_.gen.stacked4(), ref["stacked4"], rtol=1e-14, atol=0)
    np.testing.assert_allclose(sys_.zb, ref["zb"], rtol=1e-14, atol=0)
    np.testing.assert_allclose(sys_.zc, ref["zc"], rtol=1e-14, atol=0)


def test_build_excitations():
    from paper_2506_20350_b200.errors import IndexOutOfRange

    sys_ = problems.load(TBZ)
    ex = problems.build_excitations(sys_, feed_index=2)
    assert ex.matrix.shape == (sys_.dim, 6) and ex.columns == 6
    assert ex.matrix.sum() == 6 and ex.matrix[2, 0] == 1 and ex.matrix[4 + 2, 1] == 1
    with pytest.raises(IndexOutOfRange):
        problems.build_excitations(sys_, feed_index=4)
