"""Debug: the emulated peer matvec loop of test_peer_exchange_matvec_emulated, optionally synchronised."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.distributed import DeviceSlabStages, PeerExchange, _device_view, row_range, slab_ranges  # noqa
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, precompute_spectral  # noqa

ny, nx, nb, world, w, sync = [int(v) for v in sys.argv[1:7]]
gen = generator_from_stacked(seeded_stacked4(ny, nx, nb, seed=4))
op_full = precompute_spectral(gen)
st = [DeviceSlabStages(gen, world, r, torch.complex128) for r in range(world)]
l1 = st[0].l1
inner = nb * w
rows = [row_range(ny, world, r) for r in range(world)]
slabs = [slab_ranges(l1, world, r) for r in range(world)]
dev = torch.device("cuda", 0)
ex = [PeerExchange((ny * (k1 - k0) * inner, (y1 - y0) * l1 * inner), 16, dev) for (k0, k1), (y0, y1) in zip(slabs, rows)]
peers = [(e.base, e.off1, e.off2) for e in ex]
for r in range(world):
    ex[r].bind(r, world, ny, l1, inner, peers)
S = torch.cuda.synchronize if sync else (lambda: None)
for it in range(3):
    u = torch.from_numpy(dense_rhs(gen.dim, w, seed=10 + it)).cuda()
    want = matvec(op_full, u)
    ur = u.reshape(ny, nx, inner)
    for r in range(world):
        ex[r].seq += 1
        st[r].fwd_x_peer(ur[rows[r][0]:rows[r][1]], ex[r].tables[0])
    S()
    for r in range(world):
        ex[r].wait(1)
        kxs = slabs[r][1] - slabs[r][0]
        st[r].spectral_peer(ex[r].recv(1, (ny, kxs, inner), torch.complex128), ex[r].tables[1])
    S()
    outs = []
    for r in range(world):
        ex[r].wait(2)
        ny_r = rows[r][1] - rows[r][0]
        outs.append(st[r].inv_x(ex[r].recv(2, (ny_r, l1, inner), torch.complex128)))
    got = torch.cat(outs, dim=0).reshape(gen.dim, w)
    x1 = [st[r].fwd_x(ur[rows[r][0]:rows[r][1]]) for r in range(world)]
    x1s = [torch.cat([x1[q][:, slabs[r][0]:slabs[r][1]] for q in range(world)], dim=0) for r in range(world)]
    x2s = [st[r].spectral(x1s[r]) for r in range(world)]
    x2r = [torch.cat([x2s[q][rows[r][0]:rows[r][1]] for q in range(world)], dim=1) for r in range(world)]
    coll = torch.cat([st[r].inv_x(x2r[r]) for r in range(world)], dim=0).reshape(gen.dim, w)
    print("coll vs want", float((coll - want).norm() / want.norm()), "peer vs coll", float((got - coll).norm() / coll.norm()))
    for r in range(world):
        kxs = slabs[r][1] - slabs[r][0]
        print("  r", r, "recv1", float((ex[r].recv(1, (ny, kxs, inner), torch.complex128) - x1s[r]).abs().max()),
              "recv2", float((ex[r].recv(2, (rows[r][1] - rows[r][0], l1, inner), torch.complex128) - x2r[r]).abs().max()))
    err = float((got - want).norm() / want.norm())
    cnt = [_device_view(e.base, 2, torch.int64, dev).tolist() for e in ex]
    print("it", it, "rel err", err, "counters", cnt)
