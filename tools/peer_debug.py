"""Debug: compare peer-scatter receive buffers with the collective exchange layout (one GPU)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.distributed import DeviceSlabStages, PeerExchange, row_range, slab_ranges  # noqa
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked  # noqa

ny, nx, nb, world, w = [int(v) for v in sys.argv[1:6]]
gen = generator_from_stacked(seeded_stacked4(ny, nx, nb, seed=4))
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
u = torch.from_numpy(dense_rhs(gen.dim, w, seed=10)).cuda()
ur = u.reshape(ny, nx, inner)
x1 = [st[r].fwd_x(ur[rows[r][0]:rows[r][1]]) for r in range(world)]
want1 = [torch.cat([x1[q][:, slabs[r][0]:slabs[r][1]] for q in range(world)], dim=0) for r in range(world)]
for r in range(world):
    ex[r].seq += 1
    st[r].fwd_x_peer(ur[rows[r][0]:rows[r][1]], ex[r].tables[0])
torch.cuda.synchronize()
for r in range(world):
    kxs = slabs[r][1] - slabs[r][0]
    got = ex[r].recv(1, (ny, kxs, inner), torch.complex128)
    d = (got - want1[r]).abs()
    bad = (d > 1e-9 * want1[r].abs().max()).nonzero()
    print("recv1 rank", r, "maxdiff", float(d.max()), "bad", bad.shape[0], bad[:6].tolist())
x2 = [st[r].spectral(want1[r]) for r in range(world)]
want2 = [torch.cat([x2[q][rows[r][0]:rows[r][1]] for q in range(world)], dim=1) for r in range(world)]
for r in range(world):
    ex[r].wait(1)
    kxs = slabs[r][1] - slabs[r][0]
    st[r].spectral_peer(ex[r].recv(1, (ny, kxs, inner), torch.complex128), ex[r].tables[1])
torch.cuda.synchronize()
for r in range(world):
    ny_r = rows[r][1] - rows[r][0]
    got = ex[r].recv(2, (ny_r, l1, inner), torch.complex128)
    d = (got - want2[r]).abs()
    bad = (d > 1e-9 * want2[r].abs().max()).nonzero()
    print("recv2 rank", r, "maxdiff", float(d.max()), "bad", bad.shape[0], bad[:6].tolist())
