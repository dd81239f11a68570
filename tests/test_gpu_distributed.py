"""Device stages of the multi-GPU paths on one GPU: the row / kx-slab decomposed matvec
(two simulated ranks, exchanges done by hand) and a world-size-1 SlabOperator."""

import numpy as np
import pytest
import torch

from conftest import rel_err
from paper_2506_20350_b200.distributed import DeviceSlabStages, SlabOperator, row_range, slab_ranges
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, precompute_spectral

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,world", [((6, 5, 8), 2), ((30, 30, 128), 2), ((16, 16, 64), 4)])
def test_device_slab_stages_match_matvec(dims, world):
    ny, nx, nb = dims
    gen = generator_from_stacked(seeded_stacked4(ny, nx, nb, seed=3))
    u = torch.from_numpy(dense_rhs(gen.dim, 2, seed=5)).cuda()
    want = matvec(precompute_spectral(gen), u)
    st = [DeviceSlabStages(gen, world, r, torch.complex128) for r in range(world)]
    l1 = st[0].l1
    rows = [row_range(ny, world, r) for r in range(world)]
    slabs = [slab_ranges(l1, world, r) for r in range(world)]
    inner = nb * 2
    ur = u.reshape(ny, nx, inner)
    x1 = [st[r].fwd_x(ur[rows[r][0]:rows[r][1]]) for r in range(world)]
    x1s = [torch.cat([x1[q][:, slabs[r][0]:slabs[r][1]] for q in range(world)], dim=0) for r in range(world)]
    x2s = [st[r].spectral(x1s[r]) for r in range(world)]
    x2r = [torch.cat([x2s[q][rows[r][0]:rows[r][1]] for q in range(world)], dim=1) for r in range(world)]
    got = torch.cat([st[r].inv_x(x2r[r]) for r in range(world)], dim=0).reshape(gen.dim, 2)
    assert rel_err(got.cpu().numpy(), want.cpu().numpy()) <= 1e-12


@pytest.mark.parametrize("native", [True, False])
@pytest.mark.parametrize("tag", ["none", "pk"])
def test_gmres_slab_world1_matches_native(tag, native):
    from paper_2506_20350_b200.distributed import gmres_slab
    from paper_2506_20350_b200.problems import system_from_generator, unit_feed_rhs
    from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, build_pk, solve_multi_rhs_vectorized

    gen = generator_from_stacked(seeded_stacked4(4, 4, 32, seed=0))
    sys_ = system_from_generator(gen)
    p = build_pk(sys_) if tag == "pk" else None
    b = unit_feed_rhs(4, 4, 32)
    cfg = GmresConfig(tol=1e-8, restart=30)
    x, rep = gmres_slab(SlabOperator.from_generator(gen), p, b, cfg, native=native)
    xn, rn = solve_multi_rhs_vectorized(BorderedOperator.from_system(sys_), p, b[:, None], cfg)
    assert abs(rep.iterations - rn.iterations) <= 1
    assert rel_err(x, xn[:, 0]) <= 1e-7


def test_world1_slab_operator():
    gen = generator_from_stacked(seeded_stacked4(8, 8, 64, seed=2))
    op = SlabOperator.from_generator(gen)
    u = torch.from_numpy(dense_rhs(gen.dim, 3, seed=1)).cuda()
    want = matvec(precompute_spectral(gen), u)
    assert rel_err(op.matvec_local(u).cpu().numpy(), want.cpu().numpy()) <= 1e-12
    assert abs(op.norm(u) - torch.linalg.norm(u).item()) <= 1e-10 * op.norm(u)


@pytest.mark.parametrize("dims,world,w", [((6, 5, 8), 2, 2), ((16, 16, 64), 4, 1), ((9, 7, 16), 3, 3)])
def test_peer_exchange_matvec_emulated(dims, world, w):
    """Peer-scatter stages (fused all-to-all stores + arrival counters) for `world` simulated ranks
    on one GPU: every rank's pass of an exchange runs before any rank waits on it, so no kernel
    waits on another; three matvecs in a row exercise the counter epochs and the re-armed counts."""
    from paper_2506_20350_b200.distributed import PeerExchange

    ny, nx, nb = dims
    gen = generator_from_stacked(seeded_stacked4(ny, nx, nb, seed=4))
    op_full = precompute_spectral(gen)
    st = [DeviceSlabStages(gen, world, r, torch.complex128) for r in range(world)]
    l1 = st[0].l1
    inner = nb * w
    rows = [row_range(ny, world, r) for r in range(world)]
    slabs = [slab_ranges(l1, world, r) for r in range(world)]
    dev = torch.device("cuda", 0)
    ex = [PeerExchange((ny * (k1 - k0) * inner, (y1 - y0) * l1 * inner), 16, dev)
          for (k0, k1), (y0, y1) in zip(slabs, rows)]
    peers = [(e.base, e.off1, e.off2) for e in ex]
    for r in range(world):
        ex[r].bind(r, world, ny, l1, inner, peers)
    for it in range(3):
        u = torch.from_numpy(dense_rhs(gen.dim, w, seed=10 + it)).cuda()
        want = matvec(op_full, u)
        ur = u.reshape(ny, nx, inner)
        for r in range(world):
            ex[r].seq += 1
            st[r].fwd_x_peer(ur[rows[r][0]:rows[r][1]], ex[r].tables[0])
        for r in range(world):
            ex[r].wait(1)
            kxs = slabs[r][1] - slabs[r][0]
            st[r].spectral_peer(ex[r].recv(1, (ny, kxs, inner), torch.complex128), ex[r].tables[1])
        outs = []
        for r in range(world):
            ex[r].wait(2)
            ny_r = rows[r][1] - rows[r][0]
            outs.append(st[r].inv_x(ex[r].recv(2, (ny_r, l1, inner), torch.complex128)))
        got = torch.cat(outs, dim=0).reshape(gen.dim, w)
        assert rel_err(got.cpu().numpy(), want.cpu().numpy()) <= 1e-12
        for r in range(world):  # each counter saw exactly `world` arrivals per matvec
            c = torch.empty(2, dtype=torch.int64, device=dev)
            c.copy_(_counter_view(ex[r]))
            assert c.tolist() == [world * (it + 1)] * 2
    for e in ex:
        e.close()


def _counter_view(ex):
    from paper_2506_20350_b200.distributed import _device_view

    return _device_view(ex.base, 2, torch.int64, ex.device)


def _ipc_child(handle, q):
    import ctypes

    from paper_2506_20350_b200 import _lib
    from paper_2506_20350_b200.distributed import _device_view

    torch.cuda.set_device(0)
    _lib.require_cuda()
    p = ctypes.c_void_p()
    _lib.check(_lib.lib().toep_ipc_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(p)), "ipc_open")
    v = _device_view(p.value, 1024, torch.float64, torch.device("cuda", 0))
    q.put(float(v.sum().item()))
    torch.cuda.synchronize()
    _lib.check(_lib.lib().toep_ipc_close(p), "ipc_close")


def test_ipc_handle_maps_exchange_memory_in_another_process():
    import ctypes

    import torch.multiprocessing as mp

    from paper_2506_20350_b200 import _lib
    from paper_2506_20350_b200.distributed import _device_view

    _lib.require_cuda()
    p = ctypes.c_void_p()
    _lib.check(_lib.lib().toep_peer_alloc(1024 * 8, ctypes.byref(p)), "peer_alloc")
    try:
        v = _device_view(p.value, 1024, torch.float64, torch.device("cuda", 0))
        assert float(v.abs().sum().item()) == 0.0  # zero-initialised (arrival counters start at 0)
        v.copy_(torch.arange(1024, dtype=torch.float64, device="cuda"))
        torch.cuda.synchronize()
        h = (ctypes.c_char * 64)()
        _lib.check(_lib.lib().toep_ipc_handle(p, h), "ipc_handle")
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        child = ctx.Process(target=_ipc_child, args=(bytes(h), q))
        child.start()
        got = q.get(timeout=180)
        child.join(timeout=60)
        assert child.exitcode == 0
        assert got == float(1023 * 1024 // 2)
    finally:
        _lib.lib().toep_peer_free(p)


@pytest.mark.parametrize("world", [2, 3])
def test_slab_operator_built_without_full_operator(world):
    # toep_op_create_slab transforms only the rank's level-1 frequencies: its blocks equal the
    # corresponding bins of the full operator, and it keeps D * kxs / l1 bytes resident
    s4 = seeded_stacked4(6, 7, 8, seed=4)
    full = precompute_spectral(generator_from_stacked(s4))
    dfull = full.diag_blocks.reshape(full.l2, full.l1, 8, 8)
    for r in range(world):
        st = DeviceSlabStages(torch.from_numpy(s4).cuda(), world, r, torch.complex128)
        k0, k1 = slab_ranges(full.l1, world, r)
        assert (st.k0, st.k1) == (k0, k1) and (st.l2, st.l1) == (full.l2, full.l1)
        assert st.op.resident_bytes == full.resident_bytes * (k1 - k0) // full.l1
        got = st.op.diag_blocks.reshape(full.l2, k1 - k0, 8, 8)
        assert torch.equal(got, dfull[:, k0:k1])


@pytest.mark.parametrize("dims,w", [((8, 8, 64), 3), ((30, 30, 128), 1)])
def test_native_slab_apply_world1(dims, w):
    """toep_slab_apply (level-1 DFT, NCCL all-to-all over a one-rank library communicator, slab
    step, all-to-all back, inverse level-1 DFT) against the single-GPU matvec."""
    import ctypes

    from paper_2506_20350_b200 import _lib
    from paper_2506_20350_b200.distributed import native_comm

    ny, nx, nb = dims
    gen = generator_from_stacked(seeded_stacked4(ny, nx, nb, seed=4))
    op = SlabOperator.from_generator(gen)
    comm = native_comm(None)
    comm.check()
    u = torch.from_numpy(dense_rhs(gen.dim, w, seed=2)).cuda()
    want = matvec(precompute_spectral(gen), u)
    ctx = ctypes.c_void_p()
    lib = _lib.lib()
    _lib.check(lib.toep_slab_ctx_create(op.stages.op.handle, comm.handle, w, _lib.stream_handle(), ctypes.byref(ctx)))
    try:
        got = torch.empty_like(u)
        _lib.check(lib.toep_slab_apply(ctx.value, u.data_ptr(), got.data_ptr(), w, _lib.stream_handle()))
    finally:
        lib.toep_slab_ctx_destroy(ctx.value)
    assert rel_err(got.cpu().numpy(), want.cpu().numpy()) <= 1e-12
    t = torch.arange(5, dtype=torch.float64, device="cuda")
    _lib.check(lib.toep_comm_allreduce(comm.handle, t.data_ptr(), 5, _lib.stream_handle()))
    assert t.tolist() == [0.0, 1.0, 2.0, 3.0, 4.0]  # one rank: the sum is the value
