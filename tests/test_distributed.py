"""Multi-process host logic of the multi-GPU paths on CPU (gloo, world size 2): column
sharding of multi-RHS solves and the row / kx-slab decomposed matvec with its two
all-to-all exchanges.  Local compute is injected as numpy stage doubles (built from the
oracle); the device stages are covered by the gpu tests."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2506_20350_b200.distributed import SlabOperator, column_range, row_range, solve_columns_sharded
from paper_2506_20350_b200.problems import seeded_stacked4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def spawn(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    return out


def test_ranges_partition():
    for w in (1, 7, 900):
        for world in (1, 2, 3, 8):
            spans = [column_range(w, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == w
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


# ---------------------------------------------------------------- column sharding
class _Rep:
    def __init__(self, it):
        self.iterations = it
        self.converged = True


def _oracle_solver(op, p, block, cfg, method):
    d, dims = op
    x = np.zeros(block.shape, dtype=np.complex128)
    reps = []
    for c in range(block.shape[1]):
        xc, info = oracle.gmres(lambda v: oracle.matvec(d, dims, v), None, block[:, c].numpy(), cfg.tol, 200)
        x[:, c] = xc
        reps.append(_Rep(info["iterations"]))
    return torch.from_numpy(x), reps


class _Cfg:
    tol = 1e-10
    max_iter = 200


def _columns_job(rank, world, gather="all"):
    s4 = seeded_stacked4(2, 3, 4, seed=1)
    d = oracle.precompute_spectral(s4)
    dims = (2, 3, 4, 3, 5)
    rng = np.random.default_rng(0)
    b = rng.standard_normal((24, 5)) + 1j * rng.standard_normal((24, 5))
    x, reps = solve_columns_sharded((d, dims), None, torch.from_numpy(b), _Cfg(), solver=_oracle_solver,
                                    gather=gather)
    return x.numpy(), [r.iterations for r in reps]


def _columns_job_root(rank, world):
    return _columns_job(rank, world, gather="root")


def test_column_sharding_gather_to_root_gloo():
    # default gather: only rank 0 receives X; rank 1 keeps its own column range (3 of 5 -> cols 3, 4)
    out = spawn(_columns_job_root)
    assert not isinstance(out[0], str), out[0]
    assert not isinstance(out[1], str), out[1]
    x0, its0 = out[0]
    x1, its1 = out[1]
    assert x0.shape == (24, 5) and len(its0) == 5
    assert x1.shape == (24, 2) and len(its1) == 2
    assert np.array_equal(x1, x0[:, 3:])
    assert its1 == its0[3:]


def test_column_sharding_gloo():
    out = spawn(_columns_job)
    assert not isinstance(out[0], str), out[0]
    s4 = seeded_stacked4(2, 3, 4, seed=1)
    d = oracle.precompute_spectral(s4)
    dims = (2, 3, 4, 3, 5)
    rng = np.random.default_rng(0)
    b = rng.standard_normal((24, 5)) + 1j * rng.standard_normal((24, 5))
    for r in (0, 1):
        x, its = out[r]
        assert x.shape == (24, 5) and len(its) == 5
        for c in range(5):
            xc, info = oracle.gmres(lambda v: oracle.matvec(d, dims, v), None, b[:, c], 1e-10, 200)
            assert np.allclose(x[:, c], xc, rtol=1e-12, atol=1e-14)
            assert its[c] == info["iterations"]


# ---------------------------------------------------------------- slab-decomposed matvec
class NumpyStages:
    """CPU doubles of the three local stages for a (kx0, kx1) slab of the oracle's blocks."""

    def __init__(self, s4, l2, l1, k0, k1):
        k2, k1g, n0, _ = s4.shape
        self.n2, self.n1, self.n0 = (k2 + 1) // 2, (k1g + 1) // 2, n0
        self.l2, self.l1, self.k0, self.k1 = l2, l1, k0, k1
        d = oracle.precompute_spectral(s4, l2, l1).reshape(l2, l1, n0, n0)
        self.d = d[:, k0:k1]                                    # (l2, kxs, n0, n0)

    def fwd_x(self, u):                                          # (ny, n1, inner)
        ny, n1, inner = u.shape
        pad = np.zeros((ny, self.l1, inner), dtype=np.complex128)
        pad[:, :n1] = u.numpy()
        return torch.from_numpy(np.fft.fft(pad, axis=1))

    def spectral(self, x1):                                      # (n2, kxs, inner)
        n2, kxs, inner = x1.shape
        w = inner // self.n0
        pad = np.zeros((self.l2, kxs, inner), dtype=np.complex128)
        pad[:n2] = x1.numpy()
        hat = np.fft.fft(pad, axis=0).reshape(self.l2, kxs, self.n0, w)
        prod = np.einsum("abmj,abjw->abmw", self.d, hat).reshape(self.l2, kxs, inner)
        return torch.from_numpy(np.fft.ifft(prod, axis=0)[:n2].copy())

    def inv_x(self, x2):                                         # (ny, l1, inner)
        return torch.from_numpy(np.fft.ifft(x2.numpy(), axis=1)[:, : self.n1].copy())


def _slab_job(rank, world):
    ny, nx, nb, w = 5, 3, 2, 2
    s4 = seeded_stacked4(ny, nx, nb, seed=4)
    l2, l1 = 2 * ny, 2 * nx
    from paper_2506_20350_b200.distributed import slab_ranges

    k0, k1 = slab_ranges(l1, world, rank)
    op = SlabOperator(ny, nx, nb, l2, l1, NumpyStages(s4, l2, l1, k0, k1))
    rng = np.random.default_rng(3)
    u = rng.standard_normal((ny * nx * nb, w)) + 1j * rng.standard_normal((ny * nx * nb, w))
    r0, r1 = row_range(ny, world, rank)
    lo, hi = r0 * nx * nb, r1 * nx * nb
    v_local = op.matvec_local(torch.from_numpy(u[lo:hi].copy()))
    a = torch.from_numpy(u[lo:hi].copy())
    return v_local.numpy(), (lo, hi), op.dot(a, a), op.norm(a)


def test_slab_matvec_gloo():
    out = spawn(_slab_job)
    assert not isinstance(out[0], str), out[0]
    ny, nx, nb, w = 5, 3, 2, 2
    s4 = seeded_stacked4(ny, nx, nb, seed=4)
    d = oracle.precompute_spectral(s4)
    rng = np.random.default_rng(3)
    u = rng.standard_normal((ny * nx * nb, w)) + 1j * rng.standard_normal((ny * nx * nb, w))
    want = oracle.matvec(d, (ny, nx, nb, 2 * ny - 1, 2 * nx - 1), u)
    for r in (0, 1):
        v, (lo, hi), dot, nrm = out[r]
        assert np.linalg.norm(v - want[lo:hi]) <= 1e-12 * np.linalg.norm(want)
        assert abs(dot - np.vdot(u, u)) <= 1e-10 * abs(np.vdot(u, u))
        assert abs(nrm - np.linalg.norm(u)) <= 1e-10 * np.linalg.norm(u)


def _emulate_scatter(plan, outputs, recv, shape_of):
    """Apply scatter_plan routing with numpy: outputs[r] indexed [a][o][i] (pass order)."""
    for r, (lo, parts) in plan.items():
        out = outputs[r]
        n_out, outer, inner = out.shape
        for a in range(n_out):
            q = max(j for j in range(len(parts)) if lo[j] <= a and (j + 1 == len(parts) or a < lo[j + 1]))
            off, sa, so = parts[q]
            for o in range(outer):
                start = off + a * sa + o * so
                recv[q][start:start + inner] = out[a, o]
    return [recv[q].reshape(shape_of(q)) for q in range(len(recv))]


@pytest.mark.parametrize("world,n2,l1", [(2, 6, 12), (3, 7, 16), (4, 5, 12), (8, 9, 20)])
def test_peer_scatter_plan_matches_all_to_all(world, n2, l1):
    """The peer-exchange routing tables reproduce the collective exchanges' layouts."""
    from paper_2506_20350_b200.distributed import scatter_plan, slab_ranges

    inner = 3
    rng = np.random.default_rng(world)
    rows = [row_range(n2, world, q) for q in range(world)]
    slabs = [slab_ranges(l1, world, q) for q in range(world)]
    # exchange 1: rank r's level-1 output (ny_r, l1, inner) -> slab owners (n2, kxs_q, inner)
    x1 = [rng.standard_normal(((b - a), l1, inner)) for a, b in rows]
    want1 = [np.concatenate([x1[r][:, k0:k1] for r in range(world)], axis=0) for k0, k1 in slabs]
    plan0 = {r: scatter_plan(0, r, world, n2, l1, inner) for r in range(world)}
    recv1 = [np.full(n2 * (k1 - k0) * inner, np.nan) for k0, k1 in slabs]
    got1 = _emulate_scatter(plan0, {r: x1[r].transpose(1, 0, 2) for r in range(world)}, recv1,
                            lambda q: (n2, slabs[q][1] - slabs[q][0], inner))
    for q in range(world):
        np.testing.assert_array_equal(got1[q], want1[q])
    # exchange 2: rank r's slab output (n2, kxs_r, inner) -> row owners (ny_q, l1, inner)
    x2 = [rng.standard_normal((n2, (b - a), inner)) for a, b in slabs]
    want2 = [np.concatenate([x2[r][y0:y1] for r in range(world)], axis=1) for y0, y1 in rows]
    plan1 = {r: scatter_plan(1, r, world, n2, l1, inner) for r in range(world)}
    recv2 = [np.full((y1 - y0) * l1 * inner, np.nan) for y0, y1 in rows]
    got2 = _emulate_scatter(plan1, {r: x2[r] for r in range(world)}, recv2,
                            lambda q: (rows[q][1] - rows[q][0], l1, inner))
    for q in range(world):
        np.testing.assert_array_equal(got2[q], want2[q])


def test_peer_scatter_plan_rejects_empty_ranks():
    from paper_2506_20350_b200.distributed import scatter_plan
    from paper_2506_20350_b200.errors import ShapeError

    with pytest.raises(ShapeError):
        scatter_plan(0, 0, 8, 5, 12, 4)
    with pytest.raises(ValueError):
        scatter_plan(0, 0, 9, 30, 60, 4)
