"""Break down the end-to-end (pinned host in / host out) cfg2 matvec time."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4, system_from_generator  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec  # noqa

sys_ = system_from_generator(generator_from_stacked(seeded_stacked4(30, 30, 128, 0)))
op = BorderedOperator.from_system(sys_)
spec = op.spectral
n = sys_.dim
uh = torch.from_numpy(dense_rhs(n, seed=1)[:, None]).pin_memory()
ud = uh.cuda()
oh = torch.empty_like(uh).pin_memory()
s = torch.cuda.current_stream()


def ev(fn, reps=200):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3, (time.perf_counter() - t0) / reps * 1e6


print("h2d 1.84MB       us (dev, wall): %.1f %.1f" % ev(lambda: ud.copy_(uh, non_blocking=True)))
print("d2h 1.84MB       us: %.1f %.1f" % ev(lambda: oh.copy_(ud, non_blocking=True)))
print("matvec dev       us: %.1f %.1f" % ev(lambda: matvec(spec, ud)))
print("matvec e2e       us: %.1f %.1f" % ev(lambda: matvec(spec, uh)))


def manual():
    ud.copy_(uh, non_blocking=True)
    v = matvec(spec, ud)
    oh.copy_(v, non_blocking=True)
    s.synchronize()


print("manual h2d+mv+d2h+sync us: %.1f %.1f" % ev(manual))


def manual_spin():
    ud.copy_(uh, non_blocking=True)
    v = matvec(spec, ud)
    oh.copy_(v, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    while not ev.query():
        pass


print("manual + event spin us: %.1f %.1f" % ev(manual_spin))

g = torch.cuda.CUDAGraph()
vg = None
s2 = torch.cuda.Stream()
s2.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s2):
    for _ in range(3):
        ud.copy_(uh, non_blocking=True)
        vg = matvec(spec, ud)
        oh.copy_(vg, non_blocking=True)
torch.cuda.current_stream().wait_stream(s2)
torch.cuda.synchronize()
try:
    with torch.cuda.graph(g):
        ud.copy_(uh, non_blocking=True)
        vg = matvec(spec, ud)
        oh.copy_(vg, non_blocking=True)

    def graph_spin():
        g.replay()
        e = torch.cuda.Event()
        e.record()
        while not e.query():
            pass

    print("graph + event spin us: %.1f %.1f" % ev(graph_spin))
    print("graph result ok:", bool(torch.allclose(oh, matvec(spec, uh))))
except Exception as exc:  # capture of the library's launches may be refused
    print("graph capture failed:", repr(exc)[:200])
