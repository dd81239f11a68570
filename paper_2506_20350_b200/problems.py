"""Seeded inputs of the BASELINE configurations (host side).

The BASELINE generator: for every signed block offset
(p, q), p the level-2 / row / y offset and q the level-1 / column / x offset,
loop order p outer then q inner, draw ``re = N(0,1)^{Nb x Nb}`` then
``im = N(0,1)^{Nb x Nb}`` from ``numpy.random.default_rng(seed)``; the block is
``(re + 1j*im) * exp(-1j*pi*r) / max(r, 1)`` with ``r = hypot(p, q)``, and
``T(0,0) += Nb * I``.  This is the same stream the reference's test helper
``random_complex`` (``pkg/tests/helpers.py:14-15``) consumes, so
``embed_2l(blocks, Ny, Nx, Nb)`` of the reference accepts the result unchanged.

The blocks are returned directly in the reference's circulant storage order
``stacked[p % (2Ny-1), q % (2Nx-1)]`` (``toeplitz.py:59-61,193-204``), which is
what both the device operator and the oracle consume.  The whole stream is
drawn in one call per level-2 offset: numpy's Generator fills arrays in C order,
so one ``(2Nx-1, 2, Nb, Nb)`` draw equals the per-block re/im draws of the loop.
"""

from __future__ import annotations

import ctypes
import json
import struct
from dataclasses import dataclass

import numpy as np

from .errors import ChecksumMismatch, FormatVersionMismatch, InvalidSpec

__all__ = [
    "ArrayProblemSpec",
    "generate",
    "ExcitationSet",
    "build_excitations",
    "fnv1a64",
    "save",
    "load",
    "ConfigSpec",
    "CONFIGS",
    "seeded_stacked4",
    "unit_feed_rhs",
    "dense_rhs",
    "BorderedSystem",
    "system_from_generator",
    "assemble_full",
    "DEFAULT_ORACLE_CAP",
    "seeded_system",
]


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    ny: int
    nx: int
    nb: int
    note: str = ""

    @property
    def dim(self) -> int:
        return self.ny * self.nx * self.nb


CONFIGS = {
    "cfg1": ConfigSpec("cfg1", 4, 4, 32, "parity, GMRES(30) to 1e-8"),
    "cfg2": ConfigSpec("cfg2", 30, 30, 128, "headline: matvec/s + GMRES(50) to 1e-8"),
    "cfg3": ConfigSpec("cfg3", 30, 30, 256, "900 RHS multi-RHS GEMM"),
    "cfg4": ConfigSpec("cfg4", 64, 64, 128, "large single RHS, c128 + c64"),
    "cfg5": ConfigSpec("cfg5", 16, 16, 64, "block Rybicki direct solve, 4 RHS"),
}


def seeded_stacked4(ny: int, nx: int, nb: int, seed: int = 0, dtype=np.complex128) -> np.ndarray:
    """(2ny-1, 2nx-1, nb, nb) blocks in circulant order from the BASELINE generator."""
    k2, k1 = 2 * ny - 1, 2 * nx - 1
    rng = np.random.default_rng(seed)
    out = np.empty((k2, k1, nb, nb), dtype=dtype)
    qs = np.arange(-(nx - 1), nx)
    for p in range(-(ny - 1), ny):
        draw = rng.standard_normal((k1, 2, nb, nb))
        r = np.hypot(float(p), qs.astype(np.float64))
        phase = np.exp(-1j * np.pi * r)[:, None, None]
        row = (draw[:, 0] + 1j * draw[:, 1]) * phase / np.maximum(r, 1.0)[:, None, None]
        out[p % k2, qs % k1] = row
        del draw, row
    out[0, 0] += nb * np.eye(nb)
    return out


def unit_feed_rhs(ny: int, nx: int, nb: int, columns: str = "sum") -> np.ndarray:
    """Unit excitation of the first basis function of each element.

    ``columns="sum"``: one column exciting every element (cfg1/cfg2/cfg4);
    ``columns="each"``: one column per element c with a 1 at row c*nb (cfg3).
    """
    ne = ny * nx
    if columns == "sum":
        b = np.zeros(ne * nb, dtype=np.complex128)
        b[::nb] = 1.0
        return b
    if columns == "each":
        b = np.zeros((ne * nb, ne), dtype=np.complex128)
        b[np.arange(ne) * nb, np.arange(ne)] = 1.0
        return b
    raise ValueError(columns)


def dense_rhs(n: int, w: int | None = None, seed: int = 1) -> np.ndarray:
    """Complex Gaussian vector / block from ``default_rng(seed)`` (re then im)."""
    rng = np.random.default_rng(seed)
    shape = (n,) if w is None else (n, w)
    re = rng.standard_normal(shape)
    im = rng.standard_normal(shape)
    return re + 1j * im


@dataclass(frozen=True)
class BorderedSystem:
    """Bordered array system ``[[Z_A, Z_B^T], [Z_B, Z_C]]`` (problems.py:60-77 of the reference).

    ``gen`` is the generator of Z_A (a ``toeplitz.BlockGenerator2L``); ``zb`` is
    (nb, array_dim), ``zc`` (nb, nb).  The BASELINE configurations have no
    border (nb = 0); use ``system_from_generator``.
    """

    gen: object
    zb: np.ndarray
    zc: np.ndarray
    spec: object = None

    @property
    def nb(self) -> int:
        return int(self.zb.shape[0])

    @property
    def array_dim(self) -> int:
        return int(self.gen.dim)

    @property
    def dim(self) -> int:
        return self.array_dim + self.nb


def system_from_generator(gen) -> BorderedSystem:
    """Border-free system around a generator (nb = 0)."""
    return BorderedSystem(gen, np.zeros((0, gen.dim), dtype=np.complex128), np.zeros((0, 0), dtype=np.complex128))


def seeded_system(ny: int, nx: int, nb: int, seed: int = 0) -> BorderedSystem:
    """BASELINE seeded generator wrapped as an nb = 0 system."""
    from .toeplitz import generator_from_stacked

    return system_from_generator(generator_from_stacked(seeded_stacked4(ny, nx, nb, seed)))


# ------------------------------------------------------------------ synthetic bordered problems
def _helmholtz(dist2: np.ndarray, k: float, a: float) -> np.ndarray:
    """Regularised free-space kernel e^{-ikr} / (4 pi r), r = sqrt(d^2 + a^2) (problems.py:135-137)."""
    r = np.sqrt(dist2 + a * a)
    return np.exp(-1j * k * r) / (4.0 * np.pi * r)


def _border_points(rng: np.random.Generator, nb: int, wx: float, wy: float) -> np.ndarray:
    """nb sorted arc-length positions on the rectangle [0,wx]x[0,wy], walked counter-clockwise from
    the origin: bottom, right, top (right to left), left (top to bottom) (problems.py:140-154)."""
    t = np.sort(rng.uniform(0.0, 2.0 * (wx + wy), size=nb))
    pts = np.empty((nb, 2))
    edges = np.cumsum([wx, wy, wx])
    for i, ti in enumerate(t):
        if ti < edges[0]:
            pts[i] = (ti, 0.0)
        elif ti < edges[1]:
            pts[i] = (wx, ti - wx)
        elif ti < edges[2]:
            pts[i] = (2 * wx + wy - ti, wy)
        else:
            pts[i] = (0.0, 2.0 * (wx + wy) - ti)
    return pts


def generate(spec: ArrayProblemSpec) -> BorderedSystem:
    """Deterministic bordered array problem of a spec (problems.py:157-197): per-element DOF
    offsets drawn first, border positions second; block (dr, dc) entry (m, n) is the kernel at the
    element displacement plus the DOF offset difference; Z_B couples border points to every DOF,
    Z_C border to border (+ shift I).  Raises SingularMatrix if Z_C is singular."""
    from . import numerics
    from .toeplitz import generator_from_stacked

    rng = np.random.default_rng(spec.seed)
    d, k, a = spec.pitch, spec.wavenumber, spec.regularization
    dof = rng.uniform(0.0, d, size=(spec.ne, 2))
    border = _border_points(rng, spec.nb, spec.nx * d, spec.ny * d)
    # circulant offset order 0..N-1, -(N-1)..-1 at both levels (toeplitz.py:59-61)
    off_y = np.concatenate([np.arange(spec.ny), np.arange(-(spec.ny - 1), 0)]).astype(float) * d
    off_x = np.concatenate([np.arange(spec.nx), np.arange(-(spec.nx - 1), 0)]).astype(float) * d
    ddx = dof[None, :, 0] - dof[:, None, 0]
    ddy = dof[None, :, 1] - dof[:, None, 1]
    dist2 = (off_x[None, :, None, None] + ddx[None, None]) ** 2 + (off_y[:, None, None, None] + ddy[None, None]) ** 2
    stacked4 = _helmholtz(dist2, k, a)
    stacked4[0, 0] += spec.diagonal_shift * np.eye(spec.ne)
    pos = np.empty((spec.ny, spec.nx, spec.ne, 2))
    pos[..., 0] = np.arange(spec.nx)[None, :, None] * d + dof[:, 0]
    pos[..., 1] = np.arange(spec.ny)[:, None, None] * d + dof[:, 1]
    pos = pos.reshape(spec.array_dim, 2)
    zb = _helmholtz(((border[:, None, :] - pos[None, :, :]) ** 2).sum(-1), k, a)
    zc = _helmholtz(((border[:, None, :] - border[None, :, :]) ** 2).sum(-1), k, a) + \
        spec.diagonal_shift * np.eye(spec.nb)
    if spec.nb:
        numerics.lu_factor(zc)  # invertibility check (raises SingularMatrix)
    return BorderedSystem(generator_from_stacked(stacked4), zb, zc, spec)


@dataclass
class ExcitationSet:
    """One unit-feed column per array element, border rows zero (problems.py:123-132)."""

    matrix: np.ndarray
    feed_index: int

    @property
    def columns(self) -> int:
        return self.matrix.shape[1]


def build_excitations(sys: BorderedSystem, feed_index: int = 0) -> ExcitationSet:
    """Unit excitation of DOF ``feed_index`` of every element (problems.py:208-216)."""
    from .errors import IndexOutOfRange

    ne = sys.spec.ne
    if not 0 <= feed_index < ne:
        raise IndexOutOfRange(f"feed index {feed_index} outside 0..{ne - 1}")
    m = sys.spec.elements
    v = np.zeros((sys.dim, m), dtype=np.complex128)
    v[np.arange(m) * ne + feed_index, np.arange(m)] = 1.0
    return ExcitationSet(v, feed_index)


# ------------------------------------------------------------------ TBZ1 problem files
# Container of the reference's problems.save / load (problems.py:219-322): magic, little-endian
# u32 header length, sorted-key JSON header, the c128 payload (generator blocks in circulant
# order, then Z_B and Z_C, row-major, little-endian interleaved), FNV-1a-64 of the payload.
_MAGIC = b"TBZ1\n"
_VERSION = 1


@dataclass
class ArrayProblemSpec:
    """Parameters of a bordered array problem (problems.py:56-87): ``nb`` defaults to 8*(nx+ny),
    ``regularization`` to pitch/10."""

    ny: int
    nx: int
    ne: int
    nb: int | None = None
    wavenumber: float = 3.0
    pitch: float = 1.0
    regularization: float | None = None
    diagonal_shift: float = 1.0
    seed: int = 0

    def __post_init__(self):
        if self.nb is None:
            self.nb = 8 * (self.nx + self.ny)
        if self.regularization is None:
            self.regularization = self.pitch / 10.0
        if min(self.ny, self.nx, self.ne) < 1:
            raise InvalidSpec(f"ny, nx, ne must be >= 1, got {(self.ny, self.nx, self.ne)}")
        if self.nb < 0:
            raise InvalidSpec(f"nb must be >= 0, got {self.nb}")
        if not self.pitch > 0:
            raise InvalidSpec(f"pitch must be > 0, got {self.pitch}")
        if not self.regularization > 0:
            raise InvalidSpec(f"regularization must be > 0, got {self.regularization}")

    @property
    def elements(self) -> int:
        return self.ny * self.nx

    @property
    def array_dim(self) -> int:
        return self.elements * self.ne

    @property
    def dim(self) -> int:
        return self.array_dim + self.nb


def fnv1a64(data) -> int:
    """64-bit FNV-1a (problems.py:219-224), computed by libtoepcuda (host code)."""
    from . import _lib

    buf = np.frombuffer(memoryview(data).cast("B"), dtype=np.uint8) if not isinstance(data, np.ndarray) \
        else np.ascontiguousarray(data).view(np.uint8).reshape(-1)
    out = ctypes.c_uint64()
    _lib.check(_lib.lib().toep_fnv1a64(buf.ctypes.data if buf.size else None, buf.size, ctypes.byref(out)),
               "fnv1a64")
    return int(out.value)


def _payload(sys) -> list:
    return [np.ascontiguousarray(sys.gen.stacked4(), dtype="<c16"), np.ascontiguousarray(sys.zb, dtype="<c16"),
            np.ascontiguousarray(sys.zc, dtype="<c16")]


def save(sys, path) -> None:
    """Write a TBZ1 file (problems.py:236-266); ``sys.spec`` supplies the header fields."""
    s = sys.spec
    if s is None:
        raise InvalidSpec("saving a problem file needs the system's ArrayProblemSpec (sys.spec)")
    header = {"version": _VERSION, "ny": s.ny, "nx": s.nx, "ne": s.ne, "nb": s.nb, "seed": s.seed,
              "k": s.wavenumber, "pitch": s.pitch, "a": s.regularization, "shift": s.diagonal_shift,
              "dtype": "c128", "order": "row-major", "endian": "little"}
    hb = json.dumps(header, sort_keys=True).encode("utf-8")
    parts = _payload(sys)
    payload = b"".join(p.tobytes() for p in parts)
    with open(path, "wb") as fh:
        fh.write(_MAGIC)
        fh.write(struct.pack("<I", len(hb)))
        fh.write(hb)
        fh.write(payload)
        fh.write(struct.pack("<Q", fnv1a64(payload)))


def load(path) -> BorderedSystem:
    """Read a TBZ1 file (problems.py:269-322): FormatVersionMismatch for a foreign magic or
    version, ChecksumMismatch for truncated or corrupted payloads."""
    from .toeplitz import generator_from_stacked

    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[: len(_MAGIC)] != _MAGIC:
        raise FormatVersionMismatch(f"bad magic {blob[:5]!r}")
    off = len(_MAGIC)
    if len(blob) < off + 4:
        raise ChecksumMismatch("file truncated inside header length")
    (hlen,) = struct.unpack_from("<I", blob, off)
    off += 4
    if len(blob) < off + hlen:
        raise ChecksumMismatch("file truncated inside header")
    header = json.loads(blob[off: off + hlen].decode("utf-8"))
    off += hlen
    if header.get("version") != _VERSION:
        raise FormatVersionMismatch(f"unsupported version {header.get('version')!r}")
    ny, nx, ne, nb = header["ny"], header["nx"], header["ne"], header["nb"]
    n_gen = (2 * ny - 1) * (2 * nx - 1) * ne * ne
    n_zb = nb * ny * nx * ne
    n_zc = nb * nb
    expect = (n_gen + n_zb + n_zc) * 16
    if len(blob) != off + expect + 8:
        raise ChecksumMismatch(f"payload size mismatch: have {len(blob) - off - 8} bytes, expected {expect}")
    payload = memoryview(blob)[off: off + expect]
    (stored,) = struct.unpack_from("<Q", blob, off + expect)
    if fnv1a64(payload) != stored:
        raise ChecksumMismatch("payload checksum mismatch")
    scalars = np.frombuffer(payload, dtype="<c16")
    stacked4 = scalars[:n_gen].reshape(2 * ny - 1, 2 * nx - 1, ne, ne).astype(np.complex128)
    zb = scalars[n_gen: n_gen + n_zb].reshape(nb, ny * nx * ne).astype(np.complex128)
    zc = scalars[n_gen + n_zb:].reshape(nb, nb).astype(np.complex128)
    spec = ArrayProblemSpec(ny=ny, nx=nx, ne=ne, nb=nb, wavenumber=header["k"], pitch=header["pitch"],
                            regularization=header["a"], diagonal_shift=header["shift"], seed=header["seed"])
    return BorderedSystem(generator_from_stacked(stacked4), zb, zc, spec)


DEFAULT_ORACLE_CAP = 20_000  # problems.py:50 of the reference


def assemble_full(sys: BorderedSystem, cap: int = DEFAULT_ORACLE_CAP) -> np.ndarray:
    """Dense ``[[Z_A, Z_B^T], [Z_B, Z_C]]`` on the host; refuses above the oracle cap (problems.py:200-205)."""
    from .errors import TooLargeForOracle
    from .toeplitz import assemble_dense

    if sys.dim > cap:
        raise TooLargeForOracle(f"dense assembly of dimension {sys.dim} exceeds cap {cap}")
    za = assemble_dense(sys.gen)
    return np.block([[za, sys.zb.T], [sys.zb, sys.zc]])
