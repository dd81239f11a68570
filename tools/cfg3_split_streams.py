"""cfg3 900-column solve as P concurrent column sub-batches, one host thread + CUDA stream each.

The sub-batches are independent solves; while one runs its tensor-core products another can run its
HBM-bound DFT passes / orthogonalisation sweeps.  Prints the wall time (events on the default stream
bracketing the joined streams) for P = 1, 2, 3, 4.
"""
import json, os, sys, threading
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.distributed import column_range  # noqa
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, solve_multi_rhs_sequential  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec  # noqa

gen = generator_from_stacked(seeded_stacked4(30, 30, 256, 0))
sys_ = system_from_generator(gen)
op = BorderedOperator.from_system(sys_)
W = 900
B = torch.from_numpy(unit_feed_rhs(30, 30, 256, columns="each")).cuda()
cfg = GmresConfig(tol=1e-6)
which = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4]
res = {}
x_ref = None
for parts in which:
    streams = [torch.cuda.Stream() for _ in range(parts)]
    blocks = [B[:, slice(*column_range(W, parts, r))].contiguous() for r in range(parts)]
    outs = [None] * parts

    def work(r):
        with torch.cuda.stream(streams[r]):
            outs[r] = solve_multi_rhs_sequential(op, None, blocks[r], cfg)

    def run():
        cur = torch.cuda.current_stream()
        for s in streams:
            s.wait_stream(cur)
        th = [threading.Thread(target=work, args=(r,)) for r in range(parts)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for s in streams:
            cur.wait_stream(s)

    run()  # warm: per-stream workspaces
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    x = torch.cat([o[0] for o in outs], dim=1)
    its = [r.iterations for o in outs for r in o[1]]
    if x_ref is None:
        x_ref = x
    err = float((x - x_ref).norm() / x_ref.norm())
    res[f"parts_{parts}"] = {"solve_ms": ts, "median_ms": float(np.median(ts)), "it_min_max": [min(its), max(its)],
                             "rel_diff_vs_first": err}
    print(parts, json.dumps(res[f"parts_{parts}"]), flush=True)
    del streams, blocks, outs, x
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open(os.path.join("gpurun_out", "cfg3_split_streams.json"), "w"), indent=1)
