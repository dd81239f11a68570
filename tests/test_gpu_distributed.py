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


@pytest.mark.parametrize("tag", ["none", "pk"])
def test_gmres_slab_world1_matches_native(tag):
    from paper_2506_20350_b200.distributed import gmres_slab
    from paper_2506_20350_b200.problems import system_from_generator, unit_feed_rhs
    from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, build_pk, solve_multi_rhs_vectorized

    gen = generator_from_stacked(seeded_stacked4(4, 4, 32, seed=0))
    sys_ = system_from_generator(gen)
    p = build_pk(sys_) if tag == "pk" else None
    b = unit_feed_rhs(4, 4, 32)
    cfg = GmresConfig(tol=1e-8, restart=30)
    x, rep = gmres_slab(SlabOperator.from_generator(gen), p, b, cfg)
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
