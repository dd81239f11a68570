"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_golden.py [parts...]

parts: small sweep cfg1 cfg2 cfg3 cfg4 cfg5 tbz (default: small sweep cfg1 cfg2).
It imports ``toepsolve`` read-only from ``/root/reference/pkg/src`` and calls
only the reference's public API (``embed_2l``, ``precompute_spectral``,
``matvec``, ``matvec_transpose``, ``gmres``, ``build_pk``, ``rybicki_solve``,
``assemble_level1``).  Inputs come from ``paper_2506_20350_b200.problems``
(the BASELINE seeded generator), which is plain numpy and shared by both sides.
Large outputs are stored as fixed subsamples plus projections onto seeded
probe vectors (a checksum of the whole vector) so fixtures stay small.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from toepsolve.solvers import GmresConfig, build_pk, gmres, rybicki_solve, assemble_level1  # noqa: E402
from toepsolve.solvers.bordered import BorderedOperator, bordered_matvec  # noqa: E402
from toepsolve.problems import BorderedSystem, ArrayProblemSpec  # noqa: E402
from toepsolve.toeplitz import embed_2l, matvec, matvec_transpose, precompute_spectral  # noqa: E402
from toepsolve.errors import NoConvergence  # noqa: E402

from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4, unit_feed_rhs  # noqa: E402


def to_generator(stacked4):
    k2, k1, n0, _ = stacked4.shape
    n2, n1 = (k2 + 1) // 2, (k1 + 1) // 2
    blocks = {(p, q): stacked4[p % k2, q % k1] for p in range(-(n2 - 1), n2) for q in range(-(n1 - 1), n1)}
    return embed_2l(blocks, n2, n1, n0)


def loop_generator(ny, nx, nb, seed):
    """The BASELINE generator written as the literal per-block loop."""
    rng = np.random.default_rng(seed)
    blocks = {}
    for p in range(-(ny - 1), ny):
        for q in range(-(nx - 1), nx):
            g = rng.standard_normal((nb, nb)) + 1j * rng.standard_normal((nb, nb))
            r = np.hypot(p, q)
            blocks[(p, q)] = g * np.exp(-1j * np.pi * r) / max(r, 1.0)
    blocks[(0, 0)] = blocks[(0, 0)] + nb * np.eye(nb)
    return embed_2l(blocks, ny, nx, nb)


def system_nb0(gen, spec):
    return BorderedSystem(gen, np.zeros((0, gen.dim)), np.zeros((0, 0)), spec)


PROBES = 8


def probes(n, w):
    rng = np.random.default_rng(12345)
    return rng.standard_normal((PROBES, n * w)) + 1j * rng.standard_normal((PROBES, n * w))


def summarize(prefix, v, out, stride=97):
    v2 = np.asarray(v).reshape(-1)
    out[prefix + "_norm"] = np.linalg.norm(v2)
    out[prefix + "_sub"] = v2[::stride].copy()
    out[prefix + "_proj"] = probes(v2.size, 1) @ v2


def run_gmres(op, p, b, cfg):
    try:
        x, rep = gmres(lambda v: bordered_matvec(op, v), p, b, cfg)
    except NoConvergence as exc:
        x, rep = exc.solution, exc.report
    return x, rep


def part_small(out):
    # generator equivalence: vectorised draw == literal loop
    s4 = seeded_stacked4(4, 3, 5, seed=3)
    ref = loop_generator(4, 3, 5, 3).stacked4()
    assert np.array_equal(s4, ref), "seeded_stacked4 differs from the literal loop"
    out["gen_small"] = ref
    # transpose matvec + multi-column matvec on a small seeded generator
    rng = np.random.default_rng(77)
    gen = to_generator(seeded_stacked4(3, 4, 6, seed=5))
    op = precompute_spectral(gen)
    u = rng.standard_normal((gen.dim, 3)) + 1j * rng.standard_normal((gen.dim, 3))
    out["small_u"] = u
    out["small_mv"] = matvec(op, u)
    out["small_mvt"] = matvec_transpose(op, u)
    # PK apply
    spec = ArrayProblemSpec(ny=3, nx=4, ne=6, nb=0, seed=0)
    p = build_pk(system_nb0(gen, spec))
    out["small_pk"] = p.apply(u)
    # small rybicki (level-1 blocks of a seeded generator)
    gen5 = to_generator(seeded_stacked4(4, 3, 4, seed=9))
    lvl1 = assemble_level1(gen5)
    y = rng.standard_normal((gen5.dim, 2)) + 1j * rng.standard_normal((gen5.dim, 2))
    out["ryb_small_y"] = y
    out["ryb_small_x"] = rybicki_solve(lvl1, y)


def part_sweep(out):
    """test_toeplitz.py:243-252 sweep, outputs from the reference matvec."""
    rng = np.random.default_rng(17)
    dims = []
    for i in range(30):
        n2, n1 = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        n0 = int(rng.integers(1, 9))
        blocks = {}
        for o2 in range(-(n2 - 1), n2):
            for o1 in range(-(n1 - 1), n1):
                blocks[(o2, o1)] = rng.standard_normal((n0, n0)) + 1j * rng.standard_normal((n0, n0))
        gen = embed_2l(blocks, n2, n1, n0)
        u = rng.standard_normal((gen.dim, 2)) + 1j * rng.standard_normal((gen.dim, 2))
        out[f"sweep{i}_gen"] = gen.stacked4()
        out[f"sweep{i}_u"] = u
        out[f"sweep{i}_out"] = matvec(precompute_spectral(gen), u)
        dims.append((n2, n1, n0))
    out["sweep_dims"] = np.array(dims)


def part_cfg(name, ny, nx, nb, tol, restart, out, full=False, percol=None):
    t0 = time.time()
    gen = to_generator(seeded_stacked4(ny, nx, nb, seed=0))
    spec = ArrayProblemSpec(ny=ny, nx=nx, ne=nb, nb=0, seed=0)
    sys_ = system_nb0(gen, spec)
    op = BorderedOperator.from_system(sys_)
    pk = build_pk(sys_)
    print(f"[{name}] setup {time.time() - t0:.1f}s", flush=True)
    n = gen.dim
    u = dense_rhs(n, seed=1)
    t0 = time.time()
    mv = matvec(op.spectral, u)
    print(f"[{name}] matvec {time.time() - t0:.3f}s", flush=True)
    if full:
        out["mv"] = mv
        out["u"] = u
    summarize("mv", mv, out)
    cfg = GmresConfig(tol=tol, restart=restart)
    if percol is None:
        b = unit_feed_rhs(ny, nx, nb)
        for tag, p in (("none", None), ("pk", pk)):
            t0 = time.time()
            x, rep = run_gmres(op, p, b, cfg)
            print(f"[{name}] gmres {tag}: {rep.iterations} it conv={rep.converged} "
                  f"last={rep.residual_history[-1]:.3e} final={rep.final_residual:.3e} {time.time() - t0:.1f}s",
                  flush=True)
            out[f"gm_{tag}_iters"] = rep.iterations
            out[f"gm_{tag}_hist"] = np.array(rep.residual_history)
            out[f"gm_{tag}_final"] = rep.final_residual
            out[f"gm_{tag}_conv"] = rep.converged
            if full:
                out[f"gm_{tag}_x"] = x
            summarize(f"gm_{tag}_x", x, out)
    else:
        for col in percol:
            b = np.zeros(n, dtype=np.complex128)
            b[col * nb] = 1.0
            for tag, p in (("none", None), ("pk", pk)):
                t0 = time.time()
                x, rep = run_gmres(op, p, b, cfg)
                print(f"[{name}] col {col} {tag}: {rep.iterations} it {time.time() - t0:.1f}s", flush=True)
                out[f"col{col}_{tag}_iters"] = rep.iterations
                out[f"col{col}_{tag}_hist"] = np.array(rep.residual_history)
                summarize(f"col{col}_{tag}_x", x, out)
        out["percol"] = np.array(percol)


def part_cfg5(out):
    ny = nx = 16
    nb = 64
    gen = to_generator(seeded_stacked4(ny, nx, nb, seed=0))
    lvl1 = assemble_level1(gen)
    y = dense_rhs(gen.dim, 4, seed=1)
    t0 = time.time()
    x = rybicki_solve(lvl1, y)
    print(f"[cfg5] rybicki {time.time() - t0:.1f}s", flush=True)
    op = precompute_spectral(gen)
    out["res"] = np.linalg.norm(matvec(op, x) - y) / np.linalg.norm(y)
    out["x_norm"] = np.linalg.norm(x)
    out["x_sub"] = x.reshape(-1)[::97].copy()
    out["x_proj"] = probes(x.size, 1) @ x.reshape(-1)


def part_tbz(out):
    """A small bordered problem written by the reference's own TBZ1 writer (problems.py:236-266),
    plus what the reference's loader (problems.py:269-322) reads back from it."""
    from toepsolve import problems as ref_problems

    spec = ref_problems.ArrayProblemSpec(ny=2, nx=3, ne=4, nb=5, wavenumber=2.5, pitch=1.0, seed=7)
    sys_ = ref_problems.generate(spec)
    path = os.path.join(HERE, "small.tbz")
    ref_problems.save(sys_, path)
    back = ref_problems.load(path)
    out["stacked4"] = back.gen.stacked4()
    out["zb"] = back.zb
    out["zc"] = back.zc
    out["spec"] = np.array([back.spec.ny, back.spec.nx, back.spec.ne, back.spec.nb, back.spec.seed])
    out["spec_f"] = np.array([back.spec.wavenumber, back.spec.pitch, back.spec.regularization,
                              back.spec.diagonal_shift])
    with open(path, "rb") as fh:
        out["fnv"] = np.array([ref_problems.fnv1a64(fh.read()[:64])], dtype=np.uint64)


def main(parts):
    for part in parts:
        out = {}
        t0 = time.time()
        if part == "small":
            part_small(out)
        elif part == "sweep":
            part_sweep(out)
        elif part == "cfg1":
            part_cfg("cfg1", 4, 4, 32, 1e-8, 30, out, full=True)
        elif part == "cfg2":
            part_cfg("cfg2", 30, 30, 128, 1e-8, 50, out)
        elif part == "cfg4":
            part_cfg("cfg4", 64, 64, 128, 1e-6, 50, out)
        elif part == "cfg3":
            part_cfg("cfg3", 30, 30, 256, 1e-6, None, out, percol=[0, 1, 449, 899])
        elif part == "cfg5":
            part_cfg5(out)
        elif part == "tbz":
            part_tbz(out)
        else:
            raise SystemExit(f"unknown part {part}")
        path = os.path.join(HERE, f"{part}.npz")
        np.savez_compressed(path, **out)
        print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB, {time.time() - t0:.1f}s)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["small", "sweep", "cfg1", "cfg2"])
