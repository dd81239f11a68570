"""cfg3 (30x30, N_b=256, 900 unit right-hand sides): one rank's share of an N-rank column-sharded
solve, timed on one GPU for N = 1, 2, 4, 8.

The columns are independent (`distributed.solve_columns_sharded`: no data-path collective, X gathered
to rank 0 afterwards), so the device time of an N-GPU job is the time of its largest share; running
that share alone on one GPU measures it.  The line gives, per N, the share's multi-RHS matvec and
batched GMRES(1e-6) times and the job throughput W / t(share) they imply.
"""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.distributed import column_range  # noqa
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, solve_multi_rhs_sequential  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec  # noqa


def ev_time(fn, reps=1):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


gen = generator_from_stacked(seeded_stacked4(30, 30, 256, 0))
sys_ = system_from_generator(gen)
op = BorderedOperator.from_system(sys_)
W = 900
B = torch.from_numpy(unit_feed_rhs(30, 30, 256, columns="each")).cuda()
cfg = GmresConfig(tol=1e-6)
res = {}
for n in (1, 2, 4, 8):
    # the largest share of the N-rank split (rank 0 gets the remainder columns first)
    c0, c1 = max((column_range(W, n, r) for r in range(n)), key=lambda c: c[1] - c[0])
    b = B[:, c0:c1].contiguous()
    matvec(op.spectral, b)
    mv, _ = ev_time(lambda: matvec(op.spectral, b), 3)
    for _ in range(2):  # warm: per-width workspaces, allocator growth
        solve_multi_rhs_sequential(op, None, b, cfg)
    ts = []
    for _ in range(3):
        t, (x, reps) = ev_time(lambda: solve_multi_rhs_sequential(op, None, b, cfg))
        ts.append(t)
    t = float(np.min(ts))  # best of 3 after two warm-ups (the first solves at a new width allocate)
    its = [r.iterations for r in reps]
    res[f"ranks_{n}"] = {"columns_of_largest_share": c1 - c0, "matvec_ms": mv, "solve_ms": t,
                         "job_columns_per_s": W / (t * 1e-3), "it_min_max": [min(its), max(its)]}
    print(n, json.dumps(res[f"ranks_{n}"]), flush=True)
    del b, x
    torch.cuda.empty_cache()
base = res["ranks_1"]["solve_ms"]
for n in (2, 4, 8):
    res[f"ranks_{n}"]["speedup_vs_one_rank"] = base / res[f"ranks_{n}"]["solve_ms"]
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open(os.path.join("gpurun_out", "cfg3_shares.json"), "w"), indent=1)
print(json.dumps(res))
